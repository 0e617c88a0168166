# e2e (pipelined, packed per-step host buffer) x2
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe"
for i in 1 2; do
timeout 600 python bench.py $F --json-out gpurun_out/e2e_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/e2e_ab.json'));print(round(d['ms_per_step'],4),round(d['e2e']['value']/1e6,1),round(d['e2e']['ms_per_step'],4),round(d['e2e']['host_enqueue_ms_per_step'],4),round(d['e2e']['synchronous']['value']/1e6,1))"
done
nproc; uptime

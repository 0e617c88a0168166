# the config-3 step with and without the 256-MiB L2 flush between timed steps (the store is 16.5 GB > L2)
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2; do
for v in "--l2-flush" "--no-l2-flush"; do
timeout 600 python bench.py $F $v --json-out gpurun_out/flush_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/flush_ab.json'));print('$v',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"
done; done

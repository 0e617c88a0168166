F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2; do
for lf in 0.3 0.4 0.5 0.7; do
timeout 600 python bench.py $F --lf $lf --json-out gpurun_out/r02_lf.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/r02_lf.json'));print('lf $lf',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()},d['store']['bytes_device']//2**20,'MiB', d['static_recompute_ms'])"
done; done

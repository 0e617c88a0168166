# seeded tree calls (batch prologue inside the insert / delete kernels): parity, then same-box A/B
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_store.py tests/test_gpu_edge_cases.py -x -q > gpurun_out/pytest_seed.log 2>&1; echo t=$?
tail -3 gpurun_out/pytest_seed.log
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-per-tree"
for i in 1 2 3; do
timeout 900 python bench.py $F --no-seed --json-out gpurun_out/bs_a$i.json > /dev/null 2>&1
timeout 900 python bench.py $F --seed --json-out gpurun_out/bs_b$i.json > /dev/null 2>&1
for m in a b; do python -c "import json;d=json.load(open('gpurun_out/bs_$m$i.json'));print('$m',round(d['value']/1e6,1),round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['per_call_ms'].items()},round(d['e2e']['value']/1e6,1))"; done
done

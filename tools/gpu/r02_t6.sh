timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_contract.py tests/test_gpu_edge_cases.py tests/test_gpu_vanilla.py tests/test_gpu_dist.py -q -x > gpurun_out/r02_pytest6.log 2>&1; echo pytest=$?
tail -4 gpurun_out/r02_pytest6.log
timeout 600 python tools/diag_fused.py --steps 3 > gpurun_out/r02_diag_fused6.txt 2>&1; echo diag=$?
cat gpurun_out/r02_diag_fused6.txt
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab"
timeout 600 python bench.py $F --json-out gpurun_out/r02_bench6.json > gpurun_out/r02_bench6.log 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/r02_bench6.json'));print(d['ms_per_step'],d['per_call_ms'],d['latency_floor']['trees_dec'],d['latency_floor']['trees_inc'])"

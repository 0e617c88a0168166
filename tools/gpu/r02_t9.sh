timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_contract.py tests/test_gpu_vanilla.py tests/test_gpu_edge_cases.py -q -x > gpurun_out/r02_pytest9.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02_pytest9.log
timeout 600 python tools/diag_fused.py --steps 3 > gpurun_out/r02_diag_fused9.txt 2>&1; echo diag=$?
cat gpurun_out/r02_diag_fused9.txt
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab"
timeout 600 python bench.py $F --json-out gpurun_out/r02_bench9.json > gpurun_out/r02_bench9.log 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/r02_bench9.json'));print(d['ms_per_step'],d['per_call_ms'],d['static_recompute_ms'])"

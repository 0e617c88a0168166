timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_contract.py tests/test_gpu_edge_cases.py -q -x > gpurun_out/r02_pytest3.log 2>&1; echo pytest=$?
tail -4 gpurun_out/r02_pytest3.log
timeout 600 python tools/diag_fused.py --steps 4 > gpurun_out/r02_diag_fused.txt 2>&1; echo diag=$?
cat gpurun_out/r02_diag_fused.txt

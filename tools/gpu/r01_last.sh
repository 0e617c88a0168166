python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_tc.py -x -q > gpurun_out/pytest_last.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_last.log
timeout 1200 python bench.py --json-out gpurun_out/bench_last.json > gpurun_out/bench_last.log 2>&1; echo bench=$?

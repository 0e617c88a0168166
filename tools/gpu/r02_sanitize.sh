# round-2 sanitizers: memcheck / racecheck / synccheck on smoke (bench configuration) and the contract tests
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
mkdir -p gpurun_out/san
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/memcheck_smoke.log 2>&1; echo m_smoke=$?
timeout 1500 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python -m pytest -x -q tests/test_gpu_contract.py -k "not latency" > gpurun_out/san/memcheck_contract.log 2>&1; echo m_contract=$?
timeout 1500 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python -m pytest -x -q tests/test_gpu_tree.py -k "golden or config1" > gpurun_out/san/memcheck_tree.log 2>&1; echo m_tree=$?
timeout 1500 compute-sanitizer --tool racecheck --report-api-errors no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/racecheck_smoke.log 2>&1; echo r_smoke=$?
timeout 1500 compute-sanitizer --tool synccheck --report-api-errors no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/synccheck_smoke.log 2>&1; echo s_smoke=$?
for f in gpurun_out/san/*.log; do echo $f; tail -3 $f; done

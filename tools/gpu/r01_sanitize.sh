python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build26.log 2>&1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --report-api-errors no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke.log 2>&1; echo smoke=$?
timeout 1500 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python -m pytest -x -q tests/test_gpu_tree.py -k "golden or config1 or host_batches" > gpurun_out/san_tree.log 2>&1; echo tree=$?
timeout 1500 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python -m pytest -x -q tests/test_gpu_pagerank.py tests/test_gpu_wcc.py tests/test_gpu_tc.py -k "not scale24 and not scale20 and not rmat_dynamic" > gpurun_out/san_algos.log 2>&1; echo algos=$?
timeout 1500 compute-sanitizer --tool memcheck --report-api-errors no --print-limit 20 python -m pytest -x -q tests/test_gpu_store.py -k "random_batches and True-degree" > gpurun_out/san_store.log 2>&1; echo store=$?
tail -5 gpurun_out/san_smoke.log; tail -5 gpurun_out/san_tree.log; tail -5 gpurun_out/san_algos.log; tail -5 gpurun_out/san_store.log

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build28.log 2>&1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/race_smoke.log 2>&1; echo r1=$?
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -x -q tests/test_gpu_pagerank.py tests/test_gpu_tc.py tests/test_gpu_wcc.py tests/test_gpu_vanilla.py -k "closed or k3 or hand or golden" > gpurun_out/race_algos.log 2>&1; echo r2=$?
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -x -q tests/test_gpu_store.py -k "random_batches and True-degree" > gpurun_out/race_store.log 2>&1; echo r3=$?
for f in race_smoke race_algos race_store; do tail -4 gpurun_out/$f.log; done

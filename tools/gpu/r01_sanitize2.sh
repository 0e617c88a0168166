python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build27.log 2>&1
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sync_smoke.log 2>&1; echo s1=$?
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -x -q tests/test_gpu_store.py -k "random_batches and True-degree" > gpurun_out/sync_store.log 2>&1; echo s2=$?
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest -x -q tests/test_gpu_tc.py tests/test_gpu_wcc.py -k "k3 or random_static or hand or sparse" > gpurun_out/sync_algos.log 2>&1; echo s3=$?
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/race_smoke.log 2>&1; echo r1=$?
for f in sync_smoke sync_store sync_algos race_smoke; do tail -4 gpurun_out/$f.log; done

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build9.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_store.py -x -q > gpurun_out/pytest9.log 2>&1; echo t=$?
tail -30 gpurun_out/pytest9.log

timeout 1800 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/part2_pytest.log 2>&1; echo dist=$?
tail -5 gpurun_out/part2_pytest.log

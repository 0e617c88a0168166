# road-like grid stress: parity (single GPU + partitioned) and a timing datum at 2048 x 2048
timeout 1500 python -m pytest tests/test_gpu_tree.py -q -x -k grid > gpurun_out/grid_pytest.log 2>&1; echo tree=$?; tail -2 gpurun_out/grid_pytest.log
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x -k grid > gpurun_out/grid_dist.log 2>&1; echo dist=$?; tail -2 gpurun_out/grid_dist.log
timeout 900 python tools/grid_stress.py --side 2048 > gpurun_out/grid_stress.txt 2>&1; echo stress=$?; tail -12 gpurun_out/grid_stress.txt

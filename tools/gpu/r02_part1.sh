# partitioned engine (part.cu): multi-process parity (gloo host transport, P = 2..8; NCCL P = 1) + P=1 bench
timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/part1_pytest.log 2>&1; echo dist=$?
tail -30 gpurun_out/part1_pytest.log
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe"
timeout 900 python bench.py --partitioned $F --json-out gpurun_out/part1_bench.json > gpurun_out/part1_bench.log 2>&1; echo bench=$?
tail -5 gpurun_out/part1_bench.log

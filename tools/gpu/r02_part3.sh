timeout 1800 python -m pytest tests/test_gpu_dist.py -x -q -k "pipeline or 1-nccl or 4-gloo-12-True" > gpurun_out/part3_pytest.log 2>&1; echo dist=$?
tail -5 gpurun_out/part3_pytest.log
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe"
timeout 900 python bench.py --partitioned $F --json-out gpurun_out/part3_bench.json > gpurun_out/part3_bench.log 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/part3_bench.json'));print(d['ms_per_step'],{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"

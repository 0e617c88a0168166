timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -k "pipeline" > gpurun_out/part4_pytest.log 2>&1; echo dist=$?
tail -2 gpurun_out/part4_pytest.log
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe --no-e2e"
MEERKAT_PART_UNITS=1 timeout 900 python bench.py --partitioned $F --json-out gpurun_out/part4_units.json > gpurun_out/part4_units.log 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/part4_units.json'));print(d['ms_per_step'],{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()}, d.get('exchanges_per_decremental_call'))"

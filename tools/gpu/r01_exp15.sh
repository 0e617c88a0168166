python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build37.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests/test_gpu_wcc.py tests/test_gpu_store.py tests/test_abi.py -x -q > gpurun_out/pytest37.log 2>&1; echo t=$?
tail -15 gpurun_out/pytest37.log
timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --no-per-tree --json-out gpurun_out/b37.json > gpurun_out/b37.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/b37.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'])"

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build14.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py tests/test_gpu_store.py -x -q > gpurun_out/pytest14.log 2>&1; echo tree=$?
timeout 600 python tools/ab_query.py > gpurun_out/ab_query.log 2>&1; echo ab=$?
timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-cpu-baseline --json-out gpurun_out/bench14.json > gpurun_out/bench14.log 2>&1; echo bench=$?
tail -2 gpurun_out/pytest14.log; cat gpurun_out/ab_query.log
python -c "import json;d=json.load(open('gpurun_out/bench14.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'))"

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build17.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py -x -q > gpurun_out/pytest17a.log 2>&1; echo tree=$?
tail -5 gpurun_out/pytest17a.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_pagerank.py tests/test_gpu_store.py tests/test_gpu_vanilla.py -x -q > gpurun_out/pytest17b.log 2>&1; echo rest=$?
tail -5 gpurun_out/pytest17b.log
timeout 600 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-cpu-baseline --json-out gpurun_out/bench17.json > gpurun_out/bench17.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/bench17.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d['e2e'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'))"

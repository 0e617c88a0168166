python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build18.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py tests/test_gpu_vanilla.py -x -q > gpurun_out/pytest18.log 2>&1; echo t=$?
tail -3 gpurun_out/pytest18.log
timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-cpu-baseline --json-out gpurun_out/bench18.json > gpurun_out/bench18.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/bench18.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d['e2e']['value'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'),d['static_recompute_ms']);print(d['config4'])"

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build16.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_store.py tests/test_gpu_tree.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest16.log 2>&1; echo t=$?
timeout 900 python bench.py --no-compare --no-pagerank --no-wcc --no-tc --no-cpu-baseline --no-per-tree --json-out gpurun_out/bench16.json > gpurun_out/bench16.log 2>&1; echo b=$?
tail -3 gpurun_out/pytest16.log
python -c "import json;d=json.load(open('gpurun_out/bench16.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d['bulk_build'],d['e2e']);print({k:(v['ms'],v['insert_edges_per_s'],v['delete_edges_per_s'],v['query_edges_per_s']) for k,v in d['store_sweep']['by_batch'].items()})"

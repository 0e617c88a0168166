# experiment: build, GPU parity of the tree path, per-call diag, bench (reverse, no extras)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -x -q > gpurun_out/pytest5.log 2>&1; echo tree=$?
timeout 600 python tools/diag_tree.py > gpurun_out/diag5.log 2>&1; echo diag=$?
timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --json-out gpurun_out/bench5.json > gpurun_out/bench5.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest5.log; cat gpurun_out/diag5.log
python -c "import json;d=json.load(open('gpurun_out/bench5.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'))"

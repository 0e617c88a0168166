python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build22.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest22.log 2>&1; echo t=$?
tail -2 gpurun_out/pytest22.log
for i in 1 2; do timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench22_$i.json > gpurun_out/bench22_$i.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/bench22_$i.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'))"; done
timeout 600 python tools/diag_tree.py --batches 2 > gpurun_out/diag22.log 2>&1; cat gpurun_out/diag22.log | grep timeline

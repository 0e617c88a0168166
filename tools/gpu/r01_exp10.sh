python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build23.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_vanilla.py tests/test_gpu_dist.py -x -q > gpurun_out/pytest23.log 2>&1; echo t=$?
tail -2 gpurun_out/pytest23.log
for i in 1 2; do timeout 900 python bench.py --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench23_$i.json > gpurun_out/bench23_$i.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/bench23_$i.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'),d['alt']['ms_per_step'],d['alt']['per_call_ms']['trees_dec'])"; done

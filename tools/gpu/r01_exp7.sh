python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build19.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_dist.py tests/test_gpu_vanilla.py -x -q > gpurun_out/pytest19.log 2>&1; echo t=$?
tail -3 gpurun_out/pytest19.log
timeout 900 python bench.py --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --json-out gpurun_out/bench19.json > gpurun_out/bench19.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/bench19.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d['e2e']['value'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'),d['static_recompute_ms']);print(d['alt']['ms_per_step'], d['alt']['per_call_ms'])"
tail -2 gpurun_out/build19.log

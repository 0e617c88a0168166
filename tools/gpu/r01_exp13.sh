python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build31.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py tests/test_gpu_vanilla.py -x -q > gpurun_out/pytest31.log 2>&1; echo t=$?
tail -2 gpurun_out/pytest31.log
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e"
for i in 1 2; do timeout 900 python bench.py $F --json-out gpurun_out/b31_$i.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/b31_$i.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'),d['static_recompute_ms'])"; done
timeout 600 python tools/diag_tree.py --batches 2 > gpurun_out/diag31.log 2>&1; grep timeline gpurun_out/diag31.log

# same-box A/B of an experimental build (paper_2305_17813_b200/libmeerkat_spec.so) against the default
S=paper_2305_17813_b200/libmeerkat_spec.so
MEERKAT_SO_PATH=$S timeout 600 python -m pytest tests/test_gpu_tree.py tests/test_gpu_vanilla.py -x -q > gpurun_out/pytest32.log 2>&1; echo t=$?
tail -2 gpurun_out/pytest32.log
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e"
for i in 1 2; do
timeout 900 python bench.py $F --json-out gpurun_out/b32_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=$S timeout 900 python bench.py $F --json-out gpurun_out/b32_b$i.json > /dev/null 2>&1
for m in a b; do python -c "import json;d=json.load(open('gpurun_out/b32_$m$i.json'));print('$m',d['value'],d['ms_per_step'],d['per_call_ms'],d.get('sssp_ms_per_batch'),d.get('bfs_ms_per_batch'),d['static_recompute_ms'])"; done
done

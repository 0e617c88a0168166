# same-box A/B: block-0 tail rounds for frontiers of at most 128 / 256 items vs 64
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-per-tree --no-e2e"
for m in 128 256; do MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_tail$m.so timeout 900 python -m pytest tests/test_gpu_tree.py -x -q > gpurun_out/pytest_tail$m.log 2>&1; echo t$m=$?; done
for i in 1 2 3; do
timeout 900 python bench.py $F --json-out gpurun_out/bta_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_tail128.so timeout 900 python bench.py $F --json-out gpurun_out/bta_b$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_tail256.so timeout 900 python bench.py $F --json-out gpurun_out/bta_c$i.json > /dev/null 2>&1
for m in a b c; do python -c "import json;d=json.load(open('gpurun_out/bta_$m$i.json'));print('$m',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['per_call_ms'].items()},d['static_recompute_ms'])"; done
done

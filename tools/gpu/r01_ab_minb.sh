# same-box A/B: group update kernels compiled for 8 resident blocks per SM (32 regs) vs default (40)
S=paper_2305_17813_b200/libmeerkat_spec.so
MEERKAT_SO_PATH=$S timeout 900 python -m pytest tests/test_gpu_store.py tests/test_gpu_tree.py -x -q > gpurun_out/pytest_minb.log 2>&1; echo t=$?
tail -2 gpurun_out/pytest_minb.log
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-per-tree"
for i in 1 2 3; do
timeout 900 python bench.py $F --json-out gpurun_out/bm_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=$S timeout 900 python bench.py $F --json-out gpurun_out/bm_b$i.json > /dev/null 2>&1
for m in a b; do python -c "import json;d=json.load(open('gpurun_out/bm_$m$i.json'));print('$m',round(d['value']/1e6,1),round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['per_call_ms'].items()},round(d['e2e']['value']/1e6,1),d['clocks'])"; done
done

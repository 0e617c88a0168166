# same-box A/B: dynamic tree kernels compiled for 3 / 4 resident 512-thread blocks per SM vs 2
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-per-tree --no-e2e"
for m in 3 4; do MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_spec$m.so timeout 900 python -m pytest tests/test_gpu_tree.py -x -q > gpurun_out/pytest_tminb$m.log 2>&1; echo t$m=$?; done
for i in 1 2; do
timeout 900 python bench.py $F --json-out gpurun_out/bt_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_spec3.so timeout 900 python bench.py $F --json-out gpurun_out/bt_b$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_spec4.so timeout 900 python bench.py $F --json-out gpurun_out/bt_c$i.json > /dev/null 2>&1
for m in a b c; do python -c "import json;d=json.load(open('gpurun_out/bt_$m$i.json'));print('$m',round(d['value']/1e6,1),round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['per_call_ms'].items()},d['static_recompute_ms'])"; done
done

# A/B: update kernels launched with programmatic dependent launch (default) vs plain (libmeerkat_nopdl.so)
timeout 1500 python -m pytest tests/test_gpu_store.py tests/test_gpu_tree.py tests/test_gpu_contract.py tests/test_gpu_edge_cases.py -q -x > gpurun_out/pdl_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/pdl_pytest.log
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2 3; do
for v in "" nopdl; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 600 python bench.py $F --json-out gpurun_out/pdl_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/pdl_ab.json'));print('${v:-pdl}',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"
done; done

# A/B: frontier-size and invalid-list counters in different 128-B lines (default) vs the same line (libmeerkat_old.so)
timeout 1200 python -m pytest tests/test_gpu_tree.py tests/test_gpu_contract.py tests/test_gpu_edge_cases.py tests/test_gpu_vanilla.py -q -x > gpurun_out/ctrl_pytest.log 2>&1; echo pytest=$?
tail -2 gpurun_out/ctrl_pytest.log
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2 3; do
for v in "" old; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 600 python bench.py $F --json-out gpurun_out/ctrl_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/ctrl_ab.json'));print('${v:-split}',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"
done; done

# A/B: threads per block of the cooperative tree kernels (2 blocks per SM): 512 (default, 64 regs), 576 (56), 640 (48)
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_b640.so timeout 900 python -m pytest tests/test_gpu_tree.py -q -x > gpurun_out/block_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/block_pytest.log
for i in 1 2 3; do
for v in "" b576 b640; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 600 python bench.py $F --json-out gpurun_out/block_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/block_ab.json'));print('${v:-b512}',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"
done; done

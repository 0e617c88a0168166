# same-box A/B: thread-per-edge update kernels compiled for 4 / 8 resident blocks per SM vs default;
# plus the tree kernels at 1 block per SM (MEERKAT_LATENCY_BLOCKS_PER_SM=1, no rebuild)
F="--no-compare --no-pagerank --no-wcc --no-tc --no-cpu-baseline --no-per-tree --no-e2e"
for m in 4 8; do MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_spect$m.so MEERKAT_THREAD_UPD=1 timeout 900 python -m pytest tests/test_gpu_store.py tests/test_gpu_tree.py -x -q > gpurun_out/pytest_tminb$m.log 2>&1; echo t$m=$?; done
P="import json,sys;d=json.load(open(sys.argv[1]));c=d['config4'];s=d['store_sweep']['by_batch']['1000000'];print(sys.argv[2],round(d['ms_per_step'],4),{k:round(v,4) for k,v in c['per_call_ms'].items()},round(c['round_ms'],4),{k:round(v,4) for k,v in s['ms'].items()})"
for i in 1 2; do
timeout 900 python bench.py $F --json-out gpurun_out/bu_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_spect4.so timeout 900 python bench.py $F --json-out gpurun_out/bu_b$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_spect8.so timeout 900 python bench.py $F --json-out gpurun_out/bu_c$i.json > /dev/null 2>&1
for m in a b c; do python -c "$P" gpurun_out/bu_$m$i.json $m; done
done
F2="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-per-tree --no-e2e"
for i in 1 2; do
timeout 900 python bench.py $F2 --json-out gpurun_out/bl_a$i.json > /dev/null 2>&1
MEERKAT_LATENCY_BLOCKS_PER_SM=1 timeout 900 python bench.py $F2 --json-out gpurun_out/bl_b$i.json > /dev/null 2>&1
for m in a b; do python -c "import json;d=json.load(open('gpurun_out/bl_$m$i.json'));print('lat$m',round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['per_call_ms'].items()})"; done
done

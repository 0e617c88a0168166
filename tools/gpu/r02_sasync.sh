# A/B: the decremental scan through a per-lane cp.async ring (default, 5 slabs in flight per group) vs
# register double-buffering (3 per trip, libmeerkat_sreg.so); scan-mode parity first
timeout 1200 python -m pytest tests/test_gpu_tree.py tests/test_gpu_contract.py -q -x > gpurun_out/sasync_pytest.log 2>&1; echo pytest=$?
tail -1 gpurun_out/sasync_pytest.log
F="--frontier scan --no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe --steps 8"
for i in 1 2 3; do
for v in "" sreg; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 900 python bench.py $F --json-out gpurun_out/sasync_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/sasync_ab.json'));print('${v:-async}',round(d['ms_per_step'],4),round(d['per_call_ms']['trees_dec'],4),round(d['roofline']['frac'],3))"
done; done

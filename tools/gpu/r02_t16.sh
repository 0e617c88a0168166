F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for lf in 0.5 0.6 0.7 0.8; do
timeout 600 python bench.py $F --lf $lf --json-out gpurun_out/r02_lf.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/r02_lf.json'));print('lf $lf',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()},d['store']['bytes_device']//2**20,'MiB', d['static_recompute_ms'])"
done
S="--frontier scan --no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe --steps 10"
for v in "" su4; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 600 python bench.py $S --json-out gpurun_out/r02_s.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/r02_s.json'));print('scan $v',round(d['per_call_ms']['trees_dec'],4),d['roofline']['frac'])"
done
for v in "" pu3 pu4; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 600 python tools/ab_pagerank.py --reps 2
done

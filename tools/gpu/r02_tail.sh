# A/B: block-0 tail rounds up to 64 frontier items (default) vs 128 / 32
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2 3; do
for v in "" t128 t32; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 600 python bench.py $F --json-out gpurun_out/tail_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/tail_ab.json'));print('${v:-t64}',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"
done; done

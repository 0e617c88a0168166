# A/B: slabs in flight per group in the decremental scan and PageRank's accumulation (2 = default, 3, 4)
F="--no-per-tree --no-cpu-baseline --no-sweep --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2; do
for v in "" u3 u4; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO timeout 900 python bench.py $F --json-out gpurun_out/unroll_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/unroll_ab.json'));a=d['alt'];p=d['pagerank'];print('${v:-u2}','step',round(d['ms_per_step'],4),'scan',round(a['per_call_ms']['trees_dec'],4),round(a['roofline']['frac'],3),'pr',{k:p[k] for k in p if 'ms' in k or 'frac' in k})"
done; done

# A/B: store load factor (0.5 default) at HEAD
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2; do
for v in 0.4 0.5 0.6; do
timeout 600 python bench.py $F --lf $v --json-out gpurun_out/lf_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/lf_ab.json'));print('lf $v',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"
done; done

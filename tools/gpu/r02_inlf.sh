# A/B: load factor of the in-edge mirror (walked only by the decremental pull frontier): 0.5 (= --lf) / 0.7 / 0.9
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe"
for i in 1 2 3; do
for v in 0.5 0.7 0.9; do
timeout 600 python bench.py $F --in-lf $v --json-out gpurun_out/inlf_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/inlf_ab.json'));print('in-lf $v',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()})"
done; done

# partitioned P = 1, one unit per phase, own blocks through NCCL (the per-unit cost with an NCCL exchange)
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe --no-e2e"
MEERKAT_PART_UNITS=1 MEERKAT_PART_NCCL_SELF=1 timeout 900 python bench.py --partitioned $F --json-out gpurun_out/nself_bench.json > gpurun_out/nself_bench.log 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/nself_bench.json'));print(round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()}, d.get('exchanges_per_decremental_call'))"

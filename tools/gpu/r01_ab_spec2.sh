# timing-only A/B (the spec build's counters are wrong by design): no tests
S=paper_2305_17813_b200/libmeerkat_spec.so
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --no-per-tree"
for i in 1 2; do
timeout 900 python bench.py $F --json-out gpurun_out/b42_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=$S timeout 900 python bench.py $F --json-out gpurun_out/b42_b$i.json > /dev/null 2>&1
for m in a b; do python -c "import json;d=json.load(open('gpurun_out/b42_$m$i.json'));print('$m',d['value'],d['ms_per_step'],d['per_call_ms'])"; done
done

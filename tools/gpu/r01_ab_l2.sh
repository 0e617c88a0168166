# same-box A/B of L2 persistence windows (env only, one build)
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --no-per-tree"
for i in 1 2; do
for m in off node vmeta stamp; do
MEERKAT_L2_PERSIST=$m MEERKAT_L2_HIT=0.6 timeout 900 python bench.py $F --json-out gpurun_out/b48_$m.json > gpurun_out/b48_$m.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/b48_$m.json'));print('$m',d['value'],d['ms_per_step'],d['per_call_ms'])"
done; done
grep "L2 persist" gpurun_out/b48_node.log | head -2

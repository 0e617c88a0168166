F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --no-per-tree"
for i in 1 2; do
for wv in 1 4 8; do MEERKAT_UPD_WAVES=$wv timeout 900 python bench.py $F --json-out gpurun_out/b33_w$wv.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/b33_w$wv.json'));print('waves $wv',d['value'],d['ms_per_step'],d['per_call_ms'])"; done
done

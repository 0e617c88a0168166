# TC leg timing: current build vs the update kernels without the per-SM block targets (same box)
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-config4 --no-cpu-baseline --no-per-tree --no-e2e"
for i in 1 2; do
timeout 900 python bench.py $F --json-out gpurun_out/btc_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_spec.so timeout 900 python bench.py $F --json-out gpurun_out/btc_b$i.json > /dev/null 2>&1
for m in a b; do python -c "import json;d=json.load(open('gpurun_out/btc_$m$i.json'));t=d['tc'];print('$m',round(d['ms_per_step'],4),round(t['static_ms'],1),round(t['incremental_ms'],2),round(t['decremental_ms'],2))"; done
done

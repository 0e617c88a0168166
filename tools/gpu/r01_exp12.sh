python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build29.log 2>&1
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --no-per-tree"
for i in 1 2; do
timeout 900 python bench.py $F --json-out gpurun_out/b29_f$i.json > /dev/null 2>&1
timeout 900 python bench.py $F --no-l2-flush --json-out gpurun_out/b29_n$i.json > /dev/null 2>&1
for m in f n; do python -c "import json;d=json.load(open('gpurun_out/b29_$m$i.json'));print('$m',d['value'],d['ms_per_step'],d['per_call_ms'],d['config']['l2'][:20])"; done
done

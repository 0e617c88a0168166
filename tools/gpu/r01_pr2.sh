python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build7.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pagerank.py -x -q > gpurun_out/pytest7.log 2>&1; echo pr=$?
F="--no-compare --no-per-tree --no-e2e --no-cpu-baseline --steps 3"
timeout 900 python bench.py $F --json-out gpurun_out/bench7_u1.json > gpurun_out/bench7_u1.log 2>&1; echo u1=$?
MEERKAT_PR_UNROLL=2 timeout 900 python bench.py $F --no-sweep --json-out gpurun_out/bench7_u2.json > gpurun_out/bench7_u2.log 2>&1; echo u2=$?
tail -2 gpurun_out/pytest7.log
for f in gpurun_out/bench7_u1.json gpurun_out/bench7_u2.json; do python -c "import json,sys;d=json.load(open('$f'));p=d['pagerank'];print('$f',p['static_ms'],p['static_iterations'],p['per_iteration']['ms'],p['roofline']['frac'],p['incremental_ms'],p['decremental_ms'])"; done
python -c "import json;d=json.load(open('gpurun_out/bench7_u1.json'));print(json.dumps(d['store_sweep']['by_batch']))"

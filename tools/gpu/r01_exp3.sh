python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build15.log 2>&1
MEERKAT_THREAD_UPD=1 timeout 900 python -m pytest tests/test_gpu_store.py tests/test_gpu_tree.py tests/test_gpu_pagerank.py -x -q > gpurun_out/pytest15.log 2>&1; echo t=$?
F="--no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-cpu-baseline --no-per-tree --no-e2e"
timeout 900 python bench.py $F --json-out gpurun_out/bench15_g.json > gpurun_out/bench15_g.log 2>&1; echo bg=$?
MEERKAT_THREAD_UPD=1 timeout 900 python bench.py $F --json-out gpurun_out/bench15_t.json > gpurun_out/bench15_t.log 2>&1; echo bt=$?
MEERKAT_THREAD_UPD=1 timeout 900 python bench.py $F --steps 3 --sweep --json-out gpurun_out/bench15_ts.json > gpurun_out/bench15_ts.log 2>&1; echo bts=$?
tail -3 gpurun_out/pytest15.log
for f in g t; do python -c "import json;d=json.load(open('gpurun_out/bench15_$f.json'));print('$f',d['value'],d['ms_per_step'],d['per_call_ms'],d['bulk_build'])"; done
python -c "import json;d=json.load(open('gpurun_out/bench15_ts.json'));print({k:v['ms'] for k,v in d['store_sweep']['by_batch'].items()})"

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build38.log 2>&1
timeout 900 python -m pytest tests/test_gpu_wcc.py -x -q > gpurun_out/pytest38.log 2>&1; echo t=$?
tail -2 gpurun_out/pytest38.log
for i in 1 2; do timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --no-per-tree --json-out gpurun_out/b38.json > gpurun_out/b38.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/b38.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'])"; done

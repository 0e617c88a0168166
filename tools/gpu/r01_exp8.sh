python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build21.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tree.py -x -q > gpurun_out/pytest21.log 2>&1; echo t=$?
tail -3 gpurun_out/pytest21.log
timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-per-tree --no-cpu-baseline --json-out gpurun_out/bench21.json > gpurun_out/bench21.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/bench21.json'));print(d['value'],d['ms_per_step'],d['e2e'], d['roofline'])"

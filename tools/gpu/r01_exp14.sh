python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build36.log 2>&1
timeout 900 python -m pytest tests/test_gpu_vanilla.py tests/test_gpu_tree.py tests/test_abi.py -x -q > gpurun_out/pytest36.log 2>&1; echo t=$?
tail -3 gpurun_out/pytest36.log
timeout 900 python bench.py --no-compare --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-e2e --json-out gpurun_out/b36.json > gpurun_out/b36.log 2>&1; echo b=$?
python -c "import json;d=json.load(open('gpurun_out/b36.json'));print(d['value'],d['ms_per_step'],d['static_recompute_ms'],d['iteration_scheme1_static_ms'],d['vanilla_static_ms'])"

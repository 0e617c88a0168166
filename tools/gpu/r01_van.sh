python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build8.log 2>&1
timeout 900 python -m pytest tests/test_gpu_vanilla.py tests/test_gpu_tree.py tests/test_abi.py -x -q > gpurun_out/pytest8.log 2>&1; echo t=$?
timeout 900 python bench.py --no-compare --no-per-tree --no-sweep --no-pagerank --no-e2e --no-cpu-baseline --steps 5 --json-out gpurun_out/bench8.json > gpurun_out/bench8.log 2>&1; echo b=$?
tail -3 gpurun_out/pytest8.log
python -c "import json;d=json.load(open('gpurun_out/bench8.json'));print(d['ms_per_step'],d['static_recompute_ms'],d['vanilla_static_ms'],d['tree_overhead_vs_vanilla'])"

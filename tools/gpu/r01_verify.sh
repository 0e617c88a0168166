set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_store.py tests/test_gpu_tree.py -x -q > gpurun_out/pytest2.log 2>&1; echo pytest=$?
timeout 900 python bench.py --json-out gpurun_out/bench2.json > gpurun_out/bench2.log 2>&1; echo bench=$?
F="--steps 5 --warmup 3 --no-compare --no-per-tree --no-e2e --no-cpu-baseline --no-sweep"
timeout 900 ncu --nvtx --nvtx-include "timed_reverse/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv python bench.py $F > gpurun_out/ncu_list2.log 2>&1; echo list=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tree_(inc|dec)" --launch-skip 6 -c 2 -o gpurun_out/k_tree_full2 -f python bench.py $F > gpurun_out/ncu_full2.log 2>&1; echo full=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(insert|delete)" --launch-skip 8 -c 2 -o gpurun_out/k_upd_full2 -f python bench.py $F > gpurun_out/ncu_upd2.log 2>&1; echo upd=$?

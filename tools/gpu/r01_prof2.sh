python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build20.log 2>&1
F="--steps 5 --warmup 3 --no-compare --no-per-tree --no-e2e --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4"
timeout 900 ncu --nvtx --nvtx-include "timed_reverse/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches20.csv python bench.py $F > gpurun_out/ncu_list20.log 2>&1; echo list=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tree_(inc|dec)" --launch-skip 6 -c 2 -o gpurun_out/k_tree_full20 -f python bench.py $F > gpurun_out/ncu_full20.log 2>&1; echo full=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(insert|delete)" --launch-skip 8 -c 2 -o gpurun_out/k_upd_full20 -f python bench.py $F > gpurun_out/ncu_upd20.log 2>&1; echo upd=$?

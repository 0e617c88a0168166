python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_final.log
timeout 1200 python bench.py --json-out gpurun_out/bench_final.json > gpurun_out/bench_final.log 2>&1; echo bench=$?
F="--steps 5 --warmup 3 --no-compare --no-per-tree --no-e2e --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4"
timeout 900 ncu --nvtx --nvtx-include "timed_reverse/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py $F > /dev/null 2>&1; echo list=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tree_(inc|dec)" --launch-skip 6 -c 2 -o gpurun_out/k_tree_final -f python bench.py $F > /dev/null 2>&1; echo full=$?

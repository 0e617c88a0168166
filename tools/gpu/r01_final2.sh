python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_final2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_final2.log
timeout 1200 python bench.py --json-out gpurun_out/bench_final2.json > gpurun_out/bench_final2.log 2>&1; echo bench=$?
F="--steps 5 --warmup 3 --no-compare --no-per-tree --no-e2e --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4"
timeout 900 ncu --nvtx --nvtx-include "timed_reverse/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final2.csv python bench.py $F > /dev/null 2>&1; echo list=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(insert|delete)" --launch-skip 8 -c 2 -o gpurun_out/k_upd_final2 -f python bench.py $F > /dev/null 2>&1; echo full_upd=$?

# round-2: GPU suite, full bench line (latency floor, hashing A/B), launch list of the timed region
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_pytest2.log 2>&1; echo pytest=$?
tail -8 gpurun_out/r02_pytest2.log
timeout 1200 python bench.py --json-out gpurun_out/r02_bench2.json > gpurun_out/r02_bench2.log 2>&1; echo bench=$?
tail -c 400 gpurun_out/r02_bench2.log
F="--steps 5 --warmup 3 --no-compare --no-per-tree --no-e2e --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe"
timeout 900 ncu --nvtx --nvtx-include "timed_reverse/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py $F > /dev/null 2>&1; echo list=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tree_(inc|dec)|k_insert|k_delete" --launch-skip 12 -c 4 -o gpurun_out/r02_k -f python bench.py $F > /dev/null 2>&1; echo full=$?

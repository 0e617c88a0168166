# round-2 full evidence: smoke, GPU suite, default bench line, launch list, ncu --set full of the step's kernels
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02i_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02i_pytest.log
timeout 1500 python bench.py --json-out gpurun_out/r02i_bench.json > gpurun_out/r02i_bench.log 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/r02i_bench.json'));print(d['ms_per_step'],d['value']/1e6,d['e2e']['value']/1e6,d['per_call_ms'])"
F="--steps 5 --warmup 3 --no-compare --no-per-tree --no-e2e --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe"
timeout 900 ncu --nvtx --nvtx-include "timed_reverse/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_launches.csv python bench.py $F > /dev/null 2>&1; echo list=$?
timeout 900 ncu --nvtx --nvtx-include "timed_reverse/" --set full --import-source on --clock-control none -k regex:"k_tree_(inc|dec)|k_insert|k_delete" -c 4 -o gpurun_out/r02i_k -f python bench.py $F > /dev/null 2>&1; echo full=$?
timeout 900 python bench.py --partitioned --no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe --json-out gpurun_out/r02i_part.json > gpurun_out/r02i_part.log 2>&1; echo part=$?

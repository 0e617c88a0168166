python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_full2.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_full2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_full2.log
timeout 1200 python bench.py --json-out gpurun_out/bench_full2.json > gpurun_out/bench_full2.log 2>&1; echo bench=$?
timeout 900 python bench.py --partitioned --steps 3 --warmup 3 --json-out gpurun_out/bench_part.json > gpurun_out/bench_part.log 2>&1; echo part=$?
python -c "import json;d=json.load(open('gpurun_out/bench_part.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'])"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
tail -1 gpurun_out/bench_ref.log | cut -c1-300

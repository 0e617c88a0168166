python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build39.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest39.log 2>&1; echo t=$?
tail -15 gpurun_out/pytest39.log
timeout 900 python bench.py --partitioned --steps 3 --warmup 3 --json-out gpurun_out/bench_part39.json > gpurun_out/bench_part39.log 2>&1; echo part=$?
python -c "import json;d=json.load(open('gpurun_out/bench_part39.json'));print(d['value'],d['ms_per_step'],d['per_call_ms'])"
timeout 600 python tools/diag_dist.py > gpurun_out/diag39.log 2>&1; tail -6 gpurun_out/diag39.log

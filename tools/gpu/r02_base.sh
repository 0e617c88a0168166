# round-2: smoke, GPU suite, default bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest.log 2>&1; echo pytest=$?
tail -15 gpurun_out/r02_pytest.log
timeout 900 python bench.py --json-out gpurun_out/r02_bench_base.json > gpurun_out/r02_bench_base.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/r02_bench_base.log

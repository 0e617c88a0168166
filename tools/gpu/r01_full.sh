# round-end style run: build, smoke, full GPU suite, default bench, launch list of the timed region
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_full.log 2>&1; echo pytest=$?
timeout 1200 python bench.py --json-out gpurun_out/bench_full.json > gpurun_out/bench_full.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest_full.log

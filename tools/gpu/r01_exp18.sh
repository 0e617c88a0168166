python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build43.log 2>&1
timeout 900 python bench.py --partitioned --steps 3 --warmup 3 --json-out gpurun_out/bench_part43.json > gpurun_out/bench_part43.log 2>&1; echo part=$?
tail -3 gpurun_out/bench_part43.log | cut -c1-3000

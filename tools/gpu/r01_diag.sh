python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build4.log 2>&1
timeout 600 python tools/diag_tree.py > gpurun_out/diag_tree.log 2>&1; echo diag=$?
timeout 900 python bench.py --no-compare --no-per-tree --no-sweep --json-out gpurun_out/bench_pr.json > gpurun_out/bench_pr.log 2>&1; echo bench=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pagerank -c 1 -o gpurun_out/k_pagerank_full -f python bench.py --steps 3 --warmup 3 --no-compare --no-per-tree --no-sweep --no-e2e --no-cpu-baseline > gpurun_out/ncu_pr.log 2>&1; echo ncu=$?
cat gpurun_out/diag_tree.log

set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_pagerank.py -x -q > gpurun_out/pytest_pr.log 2>&1; echo pr=$?
timeout 900 python -m pytest tests/test_gpu_store.py tests/test_gpu_tree.py -x -q > gpurun_out/pytest3.log 2>&1; echo rest=$?
tail -30 gpurun_out/pytest_pr.log

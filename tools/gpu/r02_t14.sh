timeout 900 python -m pytest tests/test_gpu_pagerank.py tests/test_gpu_edge_cases.py -q -x > gpurun_out/r02_pytest14.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02_pytest14.log
for i in 1 2; do
timeout 600 python tools/ab_pagerank.py
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_c64.so timeout 600 python tools/ab_pagerank.py
done

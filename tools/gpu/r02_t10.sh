timeout 900 python -m pytest tests/test_gpu_pagerank.py -q -x > gpurun_out/r02_pytest10.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02_pytest10.log
for i in 1 2; do
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_nohint.so timeout 600 python tools/ab_pagerank.py
timeout 600 python tools/ab_pagerank.py
done

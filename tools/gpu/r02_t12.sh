timeout 900 python -m pytest tests/test_gpu_pagerank.py -q -x > gpurun_out/r02_pytest12.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02_pytest12.log
for i in 1 2; do
timeout 600 python tools/ab_pagerank.py
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_nobulk.so timeout 600 python tools/ab_pagerank.py
done
for sc in 20 22 23 24; do timeout 600 python tools/big_batch.py --scale $sc --batch 1000000; done

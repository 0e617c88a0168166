for i in 1 2; do
timeout 600 python tools/ab_pagerank.py
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_h1.so timeout 600 python tools/ab_pagerank.py
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_h2.so timeout 600 python tools/ab_pagerank.py
done
timeout 600 python tools/big_batch.py --scale 24 --batch 10000000
timeout 600 python tools/big_batch.py --scale 24 --batch 1000000
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_insert_t|k_delete_t" --launch-skip 1 -c 2 -o gpurun_out/r02_bigbatch -f python tools/big_batch.py --scale 24 --batch 10000000 > gpurun_out/r02_bigbatch_ncu.log 2>&1; echo ncu=$?

MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_diag.so timeout 600 python tools/diag_fused.py --steps 2 > gpurun_out/r02_diag5.txt 2>&1; echo diag=$?
grep -v "^DIAG" gpurun_out/r02_diag5.txt | head -20
grep "^DIAG" gpurun_out/r02_diag5.txt | tail -60

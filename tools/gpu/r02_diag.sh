# per-round group busy-time histograms of the fused seeded tree calls (diagnostics build)
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_diag.so timeout 600 python tools/diag_fused.py --steps 2 > gpurun_out/diag_rounds.txt 2>&1; echo diag=$?
timeout 600 python tools/diag_fused.py --steps 3 > gpurun_out/diag_fused_spec.txt 2>&1; echo fused=$?

# same-box A/B: k_pagerank compiled for 3 / 4 resident 512-thread blocks per SM vs 2
F="--no-compare --no-sweep --no-wcc --no-tc --no-config4 --no-cpu-baseline --no-per-tree --no-e2e"
for m in 3 4; do MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_pr$m.so timeout 900 python -m pytest tests/test_gpu_pagerank.py -x -q > gpurun_out/pytest_pr$m.log 2>&1; echo t$m=$?; done
for i in 1 2; do
timeout 900 python bench.py $F --json-out gpurun_out/bpr_a$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_pr3.so timeout 900 python bench.py $F --json-out gpurun_out/bpr_b$i.json > /dev/null 2>&1
MEERKAT_SO_PATH=paper_2305_17813_b200/libmeerkat_pr4.so timeout 900 python bench.py $F --json-out gpurun_out/bpr_c$i.json > /dev/null 2>&1
for m in a b c; do python -c "import json;d=json.load(open('gpurun_out/bpr_$m$i.json'));p=d['pagerank'];print('$m',round(p['static_ms'],2),p['static_iterations'],round(p['incremental_ms'],2),round(p['roofline']['frac'],3))"; done
done

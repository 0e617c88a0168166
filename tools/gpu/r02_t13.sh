timeout 900 python -m pytest tests/test_gpu_tree.py -q -x -k "scan or not reverse" > gpurun_out/r02_pytest13.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02_pytest13.log
F="--frontier scan --no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-e2e --no-probe --steps 10"
for i in 1 2; do
timeout 600 python bench.py $F --json-out gpurun_out/r02_scan_bulk.json > /dev/null 2>&1; python -c "import json;d=json.load(open('gpurun_out/r02_scan_bulk.json'));print('bulk',d['ms_per_step'],d['per_call_ms'],d['roofline']['frac'])"
MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_scanreg.so timeout 600 python bench.py $F --json-out gpurun_out/r02_scan_reg.json > /dev/null 2>&1; python -c "import json;d=json.load(open('gpurun_out/r02_scan_reg.json'));print('reg ',d['ms_per_step'],d['per_call_ms'],d['roofline']['frac'])"
done

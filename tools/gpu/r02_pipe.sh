# A/B: units in flight before the host reads a mode word (PIPE 2 default; 1; 4), one unit per phase at P = 1
F="--no-compare --no-per-tree --no-cpu-baseline --no-sweep --no-pagerank --no-wcc --no-tc --no-config4 --no-hashing-ab --no-probe --no-e2e"
MEERKAT_PART_UNITS=1 timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -k "pipeline" > gpurun_out/pipe_pytest.log 2>&1; echo pytest=$?
for i in 1 2; do
for v in "" pipe1 pipe4; do
if [ -z "$v" ]; then SO=""; else SO="MEERKAT_SO_PATH=$PWD/paper_2305_17813_b200/libmeerkat_$v.so"; fi
env $SO MEERKAT_PART_UNITS=1 timeout 900 python bench.py --partitioned $F --json-out gpurun_out/pipe_ab.json > /dev/null 2>&1
python -c "import json;d=json.load(open('gpurun_out/pipe_ab.json'));print('${v:-pipe2}',round(d['ms_per_step'],4),{k:round(x*1e3,1) for k,x in d['per_call_ms'].items()}, d.get('exchanges_per_decremental_call'))"
done; done

timeout 1500 python bench.py --json-out gpurun_out/r02j_bench.json > gpurun_out/r02j_bench.log 2>&1; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/r02j_bench.json'));print(d['ms_per_step'],d['value']/1e6,d['e2e']['value']/1e6,d['per_call_ms'])"

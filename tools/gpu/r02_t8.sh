free -g | head -2; nproc
timeout 2400 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > gpurun_out/r02_pytest8.log 2>&1; echo pytest=$?
tail -5 gpurun_out/r02_pytest8.log
AVAIL=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
echo avail_gb=$AVAIL
if [ "$AVAIL" -gt 150 ]; then
  timeout 2400 python tools/config5.py --json-out gpurun_out/r02_config5.json > gpurun_out/r02_config5.log 2>&1; echo config5=$?
  tail -c 1500 gpurun_out/r02_config5.log
fi

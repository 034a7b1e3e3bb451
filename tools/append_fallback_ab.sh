# APPEND overflow fallback on the device (default) vs the host-side check (HIPER_APPEND_HOST_SYNC=1):
# pooled / rerank / full-size tests, then same-box two-stage bench (device and e2e)
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_pooled.py tests/test_gpu_rerank.py tests/test_gpu_fullsize_prod.py tests/test_gpu_debug_build.py -q -p no:cacheprovider -x > gpurun_out/pytest_af.log 2>&1; tail -1 gpurun_out/pytest_af.log
for i in 1 2; do
  for v in "X=1" "HIPER_APPEND_HOST_SYNC=1"; do
    n=$(echo $v | tr '=' '_')
    env $v timeout 600 python bench.py --workload two_stage --no-cpu-baseline > gpurun_out/af_ts_${n}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/af_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['clocks']['sm_mhz'])"; done

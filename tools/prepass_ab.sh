# N3 two-stage / pooled: tests, then same-box A/B of the APPEND sample pre-pass list length
# (HIPER_PREPASS_KP=16 = the previous behaviour) and of the 8-slot register list for k <= 8
# (HIPER_POOLED_KP8=0 = the 16-slot list); launch list of one two-stage step.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_pooled.py tests/test_gpu_rerank.py tests/test_gpu_fullsize_prod.py -q -p no:cacheprovider -x > gpurun_out/pytest_pp.log 2>&1; tail -1 gpurun_out/pytest_pp.log
for i in 1 2; do
  timeout 600 python bench.py --workload two_stage --no-cpu-baseline --no-e2e > gpurun_out/pp_ts_new_$i.json 2>/dev/null
  HIPER_PREPASS_KP=16 timeout 600 python bench.py --workload two_stage --no-cpu-baseline --no-e2e > gpurun_out/pp_ts_old_$i.json 2>/dev/null
  timeout 600 python bench.py --workload config5 --k 8 --no-cpu-baseline --no-e2e > gpurun_out/pp_c5k8_new_$i.json 2>/dev/null
  HIPER_POOLED_KP8=0 timeout 600 python bench.py --workload config5 --k 8 --no-cpu-baseline --no-e2e > gpurun_out/pp_c5k8_old_$i.json 2>/dev/null
done
B="python bench.py --workload two_stage --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pp_launches.csv $B > /dev/null 2>&1
for f in gpurun_out/pp_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round((d.get('roofline') or {}).get('frac',0) or 0,4), d['clocks']['sm_mhz'])"; done

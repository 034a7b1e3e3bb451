# pooled kernel without (default) / with (HIPER_POOLED_LOCKSTEP=1) its L2 lockstep: pooled + rerank
# tests, then same-box A/B on config 5 (burst and sustained) and two-stage.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_pooled.py tests/test_gpu_rerank.py -q -p no:cacheprovider -x > gpurun_out/pytest_pls.log 2>&1; tail -1 gpurun_out/pytest_pls.log
for i in 1 2; do
  for v in "X=1" "HIPER_POOLED_LOCKSTEP=1"; do
    n=$(echo $v | tr '=' '_')
    env $v timeout 600 python bench.py --workload config5 --no-cpu-baseline --no-e2e > gpurun_out/pls_c5_${n}_$i.json 2>/dev/null
    env $v timeout 600 python bench.py --workload two_stage --no-cpu-baseline --no-e2e > gpurun_out/pls_ts_${n}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/pls_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

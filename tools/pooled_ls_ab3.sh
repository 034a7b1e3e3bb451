# pooled kernel: lockstep with the batched progress scan (HIPER_POOLED_LOCKSTEP=1) vs off (default),
# burst (5 steps) and sustained (120 steps), same box
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_pooled.py -q -p no:cacheprovider -x -k "topk or config5" > gpurun_out/pytest_pls3.log 2>&1; tail -1 gpurun_out/pytest_pls3.log
for i in 1 2; do
  for v in "X=1" "HIPER_POOLED_LOCKSTEP=1"; do
    n=$(echo $v | tr '=' '_')
    env $v timeout 600 python bench.py --workload config5 --no-cpu-baseline --no-e2e > gpurun_out/pl3_c5_${n}_$i.json 2>/dev/null
    env $v timeout 600 python bench.py --workload config5 --steps 120 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/pl3_c5long_${n}_$i.json 2>/dev/null
    env $v timeout 600 python bench.py --workload two_stage --no-cpu-baseline --no-e2e > gpurun_out/pl3_ts_${n}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/pl3_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

# per-K-block stage barriers in the MaxSim kernel (default where they fit) vs one per stage
# (HIPER_SPLIT_KB=0): GPU suite, then same-box A/B on config 3, 3v, config 2 and pipe stats
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for i in 1 2; do
  for v in "X=1" "HIPER_SPLIT_KB=0"; do
    n=$(echo $v | tr '=' '_')
    env $v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/skb_c3_${n}_$i.json 2>/dev/null
    env $v timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/skb_c3v_${n}_$i.json 2>/dev/null
    env $v timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e > gpurun_out/skb_c2g_${n}_$i.json 2>/dev/null
  done
done
for v in "X=1" "HIPER_SPLIT_KB=0"; do
  env $v HIPER_PIPE_STATS=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "hiper pipe" | tail -1 | sed "s/^/$v: /"
done
for f in gpurun_out/skb_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

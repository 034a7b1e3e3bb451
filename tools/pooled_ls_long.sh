# config 5 sustained (120 steps, ~2 s timed): L2 lockstep on vs off, same box
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do
  for v in "X=1" "HIPER_NO_LOCKSTEP=1"; do
    env $v timeout 600 python bench.py --workload config5 --steps 120 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/plsl_$(echo $v | tr '=' '_')_$i.json 2>/dev/null
  done
done
for f in gpurun_out/plsl_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['clocks'].get('power_w_median'))"; done

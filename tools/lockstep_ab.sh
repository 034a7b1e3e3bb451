# MaxSim config 3: pipe stats and same-box A/B of the L2 lockstep (default window 192 chunks) vs off
# and vs a wider window.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for v in "X=1" "HIPER_NO_LOCKSTEP=1" "HIPER_LOCKSTEP_WINDOW=512"; do
  env $v HIPER_PIPE_STATS=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "hiper pipe" | tail -1 | sed "s/^/$v: /"
done
for i in 1 2; do
  for v in "X=1" "HIPER_NO_LOCKSTEP=1" "HIPER_LOCKSTEP_WINDOW=512"; do
    env $v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ls_$(echo $v | tr '=' '_')_$i.json 2>/dev/null
  done
done
for f in gpurun_out/ls_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))"; done

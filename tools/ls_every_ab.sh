# MaxSim config 3: same-box A/B of the L2 lockstep publish / check interval (chunks)
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do
  for E in 256 16 64; do
    HIPER_LOCKSTEP_EVERY=$E timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/lse_${E}_$i.json 2>/dev/null
  done
done
for E in 16 64; do
  HIPER_LOCKSTEP_EVERY=$E HIPER_PIPE_STATS=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "hiper pipe" | tail -1 | sed "s/^/every $E: /"
done
for f in gpurun_out/lse_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))"; done

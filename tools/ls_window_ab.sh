# MaxSim config 3: lockstep window (chunks) with the warp-scanned check, same box
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do
  for W in 192 64 512; do
    HIPER_LOCKSTEP_WINDOW=$W timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/lsw_${W}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/lsw_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

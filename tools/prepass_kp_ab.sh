set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2 3; do
  for K in 6 8 16; do
    HIPER_PREPASS_KP=$K timeout 600 python bench.py --workload two_stage --no-cpu-baseline --no-e2e > gpurun_out/pp2_kp${K}_$i.json 2>/dev/null
  done
done
B="python bench.py --workload two_stage --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
HIPER_PREPASS_KP=8 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pp2_launches_kp8.csv $B > /dev/null 2>&1
for f in gpurun_out/pp2_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), d['clocks']['sm_mhz'])"; done

# packed MaxSim workloads (config 3v, 4v): same-box A/B of the L2 lockstep (default on) vs off
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for i in 1 2; do
  for v in "X=1" "HIPER_NO_LOCKSTEP=1"; do
    n=$(echo $v | tr '=' '_')
    env $v timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/pkl_c3v_${n}_$i.json 2>/dev/null
    env $v timeout 900 python bench.py --workload config3 --queries 64 --no-cpu-baseline --no-e2e > gpurun_out/pkl_q64_${n}_$i.json 2>/dev/null
  done
done
for f in gpurun_out/pkl_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

# L2 lockstep interval 256 (default) vs 16 on the other MaxSim workloads, same box
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/pytest_lse.log 2>&1; tail -1 gpurun_out/pytest_lse.log
for i in 1 2; do
  for E in 256 16; do
    HIPER_LOCKSTEP_EVERY=$E timeout 900 python bench.py --queries 64 --no-cpu-baseline --no-e2e > gpurun_out/lse2_q64_${E}_$i.json 2>/dev/null
    HIPER_LOCKSTEP_EVERY=$E timeout 900 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/lse2_c3v_${E}_$i.json 2>/dev/null
  done
done
for E in 256 16; do
  HIPER_LOCKSTEP_EVERY=$E timeout 1200 python bench.py --workload config4v --queries 256 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/lse2_c4v_${E}.json 2>/dev/null
done
for f in gpurun_out/lse2_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

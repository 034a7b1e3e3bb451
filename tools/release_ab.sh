# Early vs late accumulator release (HIPER_LATE_RELEASE=1 = late) in the MaxSim epilogues: parity
# tests of the MaxSim paths, then same-box A/B on several workloads; pipe stats of both.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_packed.py tests/test_gpu_grad.py tests/test_gpu_domain.py -q -p no:cacheprovider -x > gpurun_out/pytest_rel.log 2>&1; tail -1 gpurun_out/pytest_rel.log
W1="--chunks 300000 --steps 5 --warmup 3"
for i in 1 2; do
  for L in 0 1; do
    HIPER_LATE_RELEASE=$L timeout 300 python bench.py $W1 --no-cpu-baseline --no-e2e > gpurun_out/rel${L}_c3s_$i.json 2>/dev/null
    HIPER_LATE_RELEASE=$L timeout 300 python bench.py --workload config3v --chunks 300000 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/rel${L}_c3v_$i.json 2>/dev/null
    HIPER_LATE_RELEASE=$L timeout 300 python bench.py --workload config2 --no-cpu-baseline --no-e2e > gpurun_out/rel${L}_c2_$i.json 2>/dev/null
    HIPER_LATE_RELEASE=$L timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e > gpurun_out/rel${L}_c2g_$i.json 2>/dev/null
  done
done
for i in 1 2; do
  for L in 0 1; do
    HIPER_LATE_RELEASE=$L timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/rel${L}_c3_$i.json 2>/dev/null
  done
done
for L in 0 1; do
  HIPER_LATE_RELEASE=$L HIPER_PIPE_STATS=1 timeout 300 python bench.py --chunks 300000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "hiper pipe" | tail -1
done
for f in gpurun_out/rel*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))"; done

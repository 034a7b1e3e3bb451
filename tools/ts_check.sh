# TS-kernel experiment: parity under HIPER_MAXSIM_TS=1, then a same-box A/B of config3 (TS vs SS).
python __graft_entry__.py > gpurun_out/build.log 2>&1
HIPER_MAXSIM_TS=1 timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "topk or fullsize or config2 or batch_invariance or shard_merge" > gpurun_out/pytest_ts.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_ts.log
for i in 1 2; do
  HIPER_MAXSIM_TS=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 > gpurun_out/ts_ab_ts_$i.json 2> gpurun_out/ts_ab_ts_$i.err
  HIPER_MAXSIM_TS=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 2 > gpurun_out/ts_ab_ss_$i.json 2> gpurun_out/ts_ab_ss_$i.err
done
for f in gpurun_out/ts_ab_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))" 2>&1 | tail -1; done

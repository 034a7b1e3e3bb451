# N1 grad_d: doc-stationary kernel (default) vs the sort + segment gather path (HIPER_GRAD_D=seg):
# grad tests on both, same-box bench A/B, launch list of the new path.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "grad" > gpurun_out/pytest_gd.log 2>&1; tail -1 gpurun_out/pytest_gd.log
HIPER_GRAD_D=seg timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "grad" > gpurun_out/pytest_gd_seg.log 2>&1; tail -1 gpurun_out/pytest_gd_seg.log
for i in 1 2 3; do
  for v in "X=1" "HIPER_GRAD_D=seg"; do
    n=$(echo $v | tr '=' '_')
    env $v timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e > gpurun_out/gd_${n}_$i.json 2>/dev/null
  done
done
B="python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/gd_launches.csv $B > /dev/null 2>&1
for f in gpurun_out/gd_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us')"; done

# N1: grad tests + same-box A/B of the grad_q / grad_d fork (HIPER_GRAD_FORK=0 = serial)
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "grad" > gpurun_out/pytest_grad.log 2>&1; tail -1 gpurun_out/pytest_grad.log
for i in 1 2 3; do
  for F in 1 0; do
    HIPER_GRAD_FORK=$F timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline > gpurun_out/grad_fork${F}_$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/grad_fork${F}_$i.json')); print('fork=$F', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us', d['e2e']['value'] if d.get('e2e') else None)"
  done
done

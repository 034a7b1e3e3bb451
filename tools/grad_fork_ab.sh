# N1: grad tests + same-box A/B of launch variants given as "NAME:ENV=V,ENV=V" arguments
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "grad" > gpurun_out/pytest_grad.log 2>&1; tail -1 gpurun_out/pytest_grad.log
for i in 1 2 3; do
  for v in "$@"; do
    name=${v%%:*}; envs=$(echo ${v#*:} | tr ',' ' ')
    env $envs timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline > gpurun_out/grad_${name}_$i.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/grad_${name}_$i.json')); print('$name', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us', round(d['e2e']['value'],1) if d.get('e2e') else None)"
  done
done

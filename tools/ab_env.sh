# Same-box A/B of an environment switch on one workload: $1 = "VAR=value" (the B arm), $2.. = bench.py
# args.  Alternates A B A B; prints value / frac / clocks of each run.
set -x
V=$1; shift
python __graft_entry__.py > gpurun_out/build.log 2>&1
for i in 1 2; do
  env X=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/abenv_a_$i.json 2> gpurun_out/abenv_a_$i.err
  env $V timeout 900 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/abenv_b_$i.json 2> gpurun_out/abenv_b_$i.err
done
for f in gpurun_out/abenv_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))"; done

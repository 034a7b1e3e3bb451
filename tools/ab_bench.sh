# Same-box A/B of two libhiper.so builds on one workload: $1 = the other .so, $2.. = bench.py args.
# Alternates A B A B so box drift hits both; prints one JSON line per run to gpurun_out/ab_*.json.
set -x
OTHER=$1; shift
cp paper_2505_04846_b200/libhiper.so /tmp/lib_new.so
for i in 1 2; do
  cp /tmp/lib_new.so paper_2505_04846_b200/libhiper.so
  timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab_new_$i.json 2> gpurun_out/ab_new_$i.err
  cp $OTHER paper_2505_04846_b200/libhiper.so
  timeout 600 python bench.py --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab_old_$i.json 2> gpurun_out/ab_old_$i.err
done
cp /tmp/lib_new.so paper_2505_04846_b200/libhiper.so
for f in gpurun_out/ab_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"; done

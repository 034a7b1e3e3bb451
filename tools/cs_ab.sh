# Chunk-stationary pooled kernel (a12): GPU tests + same-box A/B of config 5 over variants given as
# arguments "NAME:ENV=V,ENV=V" against the streaming kernel (HIPER_POOLED_CS=0).
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
timeout 600 python -m pytest tests/test_gpu_pooled.py -q -p no:cacheprovider -x > gpurun_out/pytest_pooled.log 2>&1; echo rc=$? >> gpurun_out/pytest_pooled.log
tail -3 gpurun_out/pytest_pooled.log
fi
VARS="$* old:HIPER_POOLED_CS=0"
for i in 1 2; do
  for v in $VARS; do
    name=${v%%:*}; envs=$(echo ${v#*:} | tr ',' ' ')
    env $envs timeout 300 python bench.py --workload config5 --no-cpu-baseline > gpurun_out/c5_${name}_$i.json 2> gpurun_out/c5_${name}_$i.err
  done
done
for v in $*; do
  name=${v%%:*}; envs=$(echo ${v#*:} | tr ',' ' ')
  env $envs HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/c5_stats_$name.log
  echo $name; grep "hiper pipe" gpurun_out/c5_stats_$name.log | tail -1
done
for f in gpurun_out/c5_*.json; do python -c "import json; d=json.loads(open('$f').readline()); print('$f', round(d['value']), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done

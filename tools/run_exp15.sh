# Ablation: how much do the epilogue and the L2 feed cost?  config3 300k, HIPER_DEBUG_MODE 0..3.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for v in 0 1 2 3; do
  echo "== HIPER_DEBUG_MODE=$v" >> gpurun_out/exp15.txt
  HIPER_DEBUG_MODE=$v HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/exp15.json 2> gpurun_out/exp15.err
  grep "hiper pipe" gpurun_out/exp15.err | head -1 >> gpurun_out/exp15.txt
  python -c "import json;d=json.load(open('gpurun_out/exp15.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'],d['clocks']['power_w_median'])" >> gpurun_out/exp15.txt
done
echo all_done >> gpurun_out/exp15.txt

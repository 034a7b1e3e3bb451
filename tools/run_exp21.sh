# Wait policy, second round: try_wait without a suspend hint for the epilogue (16) / MMA (32).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for sp in 1 17 32 48 1 17; do
  echo "== HIPER_SPIN=$sp" >> gpurun_out/exp21.txt
  HIPER_SPIN=$sp HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/exp21.json 2> gpurun_out/exp21.err
  grep "hiper pipe" gpurun_out/exp21.err | head -1 >> gpurun_out/exp21.txt
  python -c "import json;d=json.load(open('gpurun_out/exp21.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/exp21.txt 2>&1
done
echo all_done >> gpurun_out/exp21.txt

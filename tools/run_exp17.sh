# Wait policy ablation: suspend (try_wait + time hint) vs busy-wait (test_wait) for the MMA thread
# (HIPER_SPIN=1) and also the epilogue (HIPER_SPIN=3), production and debug mode 2.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for m in 0 2; do for sp in 0 1 3; do
  echo "== HIPER_DEBUG_MODE=$m HIPER_SPIN=$sp" >> gpurun_out/exp17.txt
  HIPER_DEBUG_MODE=$m HIPER_SPIN=$sp HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/exp17.json 2> gpurun_out/exp17.err
  grep "hiper pipe" gpurun_out/exp17.err | head -1 >> gpurun_out/exp17.txt
  python -c "import json;d=json.load(open('gpurun_out/exp17.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/exp17.txt 2>&1
done; done
echo all_done >> gpurun_out/exp17.txt

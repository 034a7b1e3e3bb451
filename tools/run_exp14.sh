# Where do the MMA thread's full-stage waits (18%) come from?  Lockstep window / no lockstep, config3 300k.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config3 --chunks 300000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for v in "" "HIPER_LOCKSTEP_WINDOW=384" "HIPER_LOCKSTEP_WINDOW=1024" "HIPER_NO_LOCKSTEP=1" "HIPER_BAND_MB=48"; do
  echo "== $v" >> gpurun_out/exp14.txt
  env $v HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/exp14.json 2> gpurun_out/exp14.err
  grep "hiper pipe" gpurun_out/exp14.err | head -1 >> gpurun_out/exp14.txt
  python -c "import json;d=json.load(open('gpurun_out/exp14.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/exp14.txt
done
echo all_done >> gpurun_out/exp14.txt

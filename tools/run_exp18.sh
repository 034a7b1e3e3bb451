# Busy-waiting MMA thread as the default: rerank/packed tests, full-size A/B of the wait policy.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_rerank.py tests/test_gpu_packed.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_part.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_part.log
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for sp in 0 1 5; do
  echo "== HIPER_SPIN=$sp" >> gpurun_out/exp18.txt
  HIPER_SPIN=$sp HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/exp18.json 2> gpurun_out/exp18.err
  grep "hiper pipe" gpurun_out/exp18.err | head -1 >> gpurun_out/exp18.txt
  python -c "import json;d=json.load(open('gpurun_out/exp18.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/exp18.txt 2>&1
done
for sp in 0 1 0 1; do
  echo "== full config3 HIPER_SPIN=$sp" >> gpurun_out/exp18.txt
  HIPER_SPIN=$sp timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/exp18.json 2> gpurun_out/exp18.err
  python -c "import json;d=json.load(open('gpurun_out/exp18.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/exp18.txt 2>&1
done
for sp in 0 1; do
  echo "== config3v HIPER_SPIN=$sp" >> gpurun_out/exp18.txt
  HIPER_SPIN=$sp timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/exp18.json 2> gpurun_out/exp18.err
  python -c "import json;d=json.load(open('gpurun_out/exp18.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/exp18.txt 2>&1
done
echo all_done >> gpurun_out/exp18.txt

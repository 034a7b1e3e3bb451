# Software-pipelined x32 TMEM reads in the dense epilogue: parity, pipe stats and full config3 A/B.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for sp in 9 1; do
  echo "== HIPER_SPIN=$sp" >> gpurun_out/exp19.txt
  HIPER_SPIN=$sp HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/exp19.json 2> gpurun_out/exp19.err
  grep "hiper pipe" gpurun_out/exp19.err | head -1 >> gpurun_out/exp19.txt
  python -c "import json;d=json.load(open('gpurun_out/exp19.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/exp19.txt 2>&1
done
for sp in 9 1 9 1; do
  echo "== full config3 HIPER_SPIN=$sp" >> gpurun_out/exp19.txt
  HIPER_SPIN=$sp timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/exp19.json 2> gpurun_out/exp19.err
  python -c "import json;d=json.load(open('gpurun_out/exp19.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/exp19.txt 2>&1
done
echo "== config5 pooled (spin default)" >> gpurun_out/exp19.txt
timeout 600 python bench.py --workload config5 --no-cpu-baseline --no-e2e > gpurun_out/exp19.json 2> gpurun_out/exp19.err
python -c "import json;d=json.load(open('gpurun_out/exp19.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/exp19.txt 2>&1
echo "== config5 pooled HIPER_SPIN=0" >> gpurun_out/exp19.txt
HIPER_SPIN=0 timeout 600 python bench.py --workload config5 --no-cpu-baseline --no-e2e > gpurun_out/exp19.json 2> gpurun_out/exp19.err
python -c "import json;d=json.load(open('gpurun_out/exp19.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/exp19.txt 2>&1
echo all_done >> gpurun_out/exp19.txt

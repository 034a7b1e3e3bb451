# Split accumulators (4 TMEM slots of 128 columns): GPU parity suite, pipe stats split vs unsplit,
# config3 / config3v benches.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for v in "HIPER_NO_SPLIT=1" "HIPER_SPLIT_ON=1" "HIPER_DEBUG_MODE=2" "HIPER_DEBUG_MODE=3"; do
  echo "== $v" >> gpurun_out/split.txt
  env $v HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/split.json 2> gpurun_out/split.err
  grep "hiper pipe" gpurun_out/split.err | head -1 >> gpurun_out/split.txt
  python -c "import json;d=json.load(open('gpurun_out/split.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/split.txt 2>&1
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --workload config3v --no-cpu-baseline > gpurun_out/bench_c3v.json 2> gpurun_out/bench_c3v.err
echo all_done >> gpurun_out/split.txt

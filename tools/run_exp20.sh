# (1) per-chunk fixed cost: debug mode 4 (each chunk's K loop twice, no epilogue, no TMA) vs mode 2;
# (2) config2 e2e: prefetching copy stream vs serial copies, same box.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for m in 2 4; do
  echo "== HIPER_DEBUG_MODE=$m" >> gpurun_out/exp20.txt
  HIPER_DEBUG_MODE=$m HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/exp20.json 2> gpurun_out/exp20.err
  grep "hiper pipe" gpurun_out/exp20.err | head -1 >> gpurun_out/exp20.txt
done
for v in "" "--e2e-serial" "" "--e2e-serial"; do
  echo "== config2 $v" >> gpurun_out/exp20.txt
  timeout 300 python bench.py --workload config2 --no-cpu-baseline $v > gpurun_out/exp20.json 2> gpurun_out/exp20.err
  python -c "import json;d=json.load(open('gpurun_out/exp20.json'));print(d['value'],d['e2e']['value'])" >> gpurun_out/exp20.txt 2>&1
done
echo all_done >> gpurun_out/exp20.txt

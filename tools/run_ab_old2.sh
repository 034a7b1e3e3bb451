# Same-box A/B #2: session-start kernel vs current with HIPER_SPIN=0 / 1 (pipe stats, 300k chunks).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
(cd _old && python __graft_entry__.py > ../gpurun_out/build_old.log 2>&1)
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for v in old new0 new1 old new0 new1; do
  echo "== $v pipe 300k" >> gpurun_out/ab_old2.txt
  case $v in
    old) (cd _old && HIPER_PIPE_STATS=1 timeout 300 $B > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err) ;;
    new0) HIPER_SPIN=0 HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/ab.json 2> gpurun_out/ab.err ;;
    new1) HIPER_SPIN=1 HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/ab.json 2> gpurun_out/ab.err ;;
  esac
  grep "hiper pipe" gpurun_out/ab.err | head -1 >> gpurun_out/ab_old2.txt
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/ab_old2.txt 2>&1
done
echo all_done >> gpurun_out/ab_old2.txt

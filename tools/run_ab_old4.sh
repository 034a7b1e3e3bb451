# Same-box A/B #4: session-start kernel vs current (MMA busy-wait) vs current with MMA suspend (_var).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
(cd _old && python __graft_entry__.py > ../gpurun_out/build_old.log 2>&1)
(cd _var && python __graft_entry__.py > ../gpurun_out/build_var.log 2>&1)
B="python bench.py --workload config3 --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for v in old var new old var new; do
  echo "== $v pipe 300k" >> gpurun_out/ab_old4.txt
  case $v in
    old) (cd _old && HIPER_PIPE_STATS=1 timeout 300 $B > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err) ;;
    var) (cd _var && HIPER_PIPE_STATS=1 timeout 300 $B > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err) ;;
    new) HIPER_PIPE_STATS=1 timeout 300 $B > gpurun_out/ab.json 2> gpurun_out/ab.err ;;
  esac
  grep "hiper pipe" gpurun_out/ab.err | head -1 >> gpurun_out/ab_old4.txt
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/ab_old4.txt 2>&1
done
echo all_done >> gpurun_out/ab_old4.txt

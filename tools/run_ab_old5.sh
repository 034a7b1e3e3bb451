# Same-box A/B #5: session-start kernel vs current (instrumentation compiled out of production).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
(cd _old && python __graft_entry__.py > ../gpurun_out/build_old.log 2>&1)
B="python bench.py --workload config3 --chunks 300000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for v in old new old new old new; do
  echo "== $v 300k" >> gpurun_out/ab_old5.txt
  if [ $v = old ]; then (cd _old && timeout 300 $B > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 300 $B > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/ab_old5.txt 2>&1
done
for v in old new old new; do
  echo "== $v full config3" >> gpurun_out/ab_old5.txt
  if [ $v = old ]; then (cd _old && timeout 600 python bench.py --no-cpu-baseline --no-e2e > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/ab_old5.txt 2>&1
done
for v in old new; do
  echo "== $v config3v" >> gpurun_out/ab_old5.txt
  if [ $v = old ]; then (cd _old && timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/ab_old5.txt 2>&1
done
echo all_done >> gpurun_out/ab_old5.txt

# Same-box A/B: _var (previous commit, built in _var/) vs the working tree.  usage: run_ab_var.sh TAG
T=${1:-ab_var}
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
(cd _var && python __graft_entry__.py > ../gpurun_out/build_var.log 2>&1)
B="python bench.py --workload config3 --chunks 300000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for v in var new var new var new; do
  echo "== $v 300k" >> gpurun_out/$T.txt
  if [ $v = var ]; then (cd _var && timeout 300 $B > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 300 $B > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['clocks']['sm_mhz'])" >> gpurun_out/$T.txt 2>&1
done
for v in var new var new; do
  echo "== $v full config3" >> gpurun_out/$T.txt
  if [ $v = var ]; then (cd _var && timeout 600 python bench.py --no-cpu-baseline --no-e2e > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks'])" >> gpurun_out/$T.txt 2>&1
done
echo all_done >> gpurun_out/$T.txt

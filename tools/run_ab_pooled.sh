# Same-box A/B, pooled kernel (config5): _var (instrumented production build) vs working tree.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
(cd _var && python __graft_entry__.py > ../gpurun_out/build_var.log 2>&1)
cp MEASURED_PEAKS.json _var/ 2>/dev/null
for v in var new var new var new; do
  echo "== $v config5" >> gpurun_out/ab_pooled.txt
  if [ $v = var ]; then (cd _var && timeout 600 python bench.py --workload config5 --no-cpu-baseline --no-e2e > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 600 python bench.py --workload config5 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks']['sm_mhz'])" >> gpurun_out/ab_pooled.txt 2>&1
done
for v in var new; do
  echo "== $v config3v" >> gpurun_out/ab_pooled.txt
  if [ $v = var ]; then (cd _var && timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks']['sm_mhz'])" >> gpurun_out/ab_pooled.txt 2>&1
done
echo all_done >> gpurun_out/ab_pooled.txt

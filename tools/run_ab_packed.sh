# Transposed-butterfly packed pass 3: packed/rerank parity tests, then same-box A/B vs _var (HEAD).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
(cd _var && python __graft_entry__.py > ../gpurun_out/build_var.log 2>&1)
timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_rerank.py -q -x -p no:cacheprovider > gpurun_out/pytest_packed.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_packed.log
for v in var new var new var new; do
  echo "== $v config3v" >> gpurun_out/ab_packed.txt
  if [ $v = var ]; then (cd _var && timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > ../gpurun_out/ab.json 2> ../gpurun_out/ab.err);
  else timeout 600 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2> gpurun_out/ab.err; fi
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(d['value'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks']['sm_mhz'])" >> gpurun_out/ab_packed.txt 2>&1
done
echo all_done >> gpurun_out/ab_packed.txt

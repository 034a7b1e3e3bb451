set -x
bash tools/gpu_tests.sh "pooled or rerank or shard_merge or domain" || exit 1
timeout 900 python bench.py --workload two_stage --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ts_bench2.json 2> gpurun_out/ts_bench2.err
timeout 900 python bench.py --workload config5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c5_bench2.json 2> gpurun_out/c5_bench2.err
python - <<'P'
import json
for f in ["gpurun_out/ts_bench2.json", "gpurun_out/c5_bench2.json"]:
    try:
        d = json.load(open(f))
        print(f, d["value"], d["ms_per_step"], [ (s["kernel_ms_per_launch"], s["frac"]) for s in d.get("roofline_stages", [d["roofline"]])])
    except Exception as e:
        print(f, "ERR", e)
P

# pooled k > 16 heap path with the pub8 bound: tests + probe_pooled_k timings at k = 10, 100, 128
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "pooled or rerank or shard_merge" 2>&1 | tail -2
KS=10,100,128 timeout 300 python tools/probe_pooled_k.py
HIPER_NO_PUB8=1 KS=100 timeout 300 python tools/probe_pooled_k.py
HIPER_PIPE_STATS=1 KS=100 timeout 300 python tools/probe_pooled_k.py 2>&1 | grep "hiper pipe" | tail -1
timeout 600 python bench.py --workload two_stage --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ts_bench3.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/ts_bench3.json')); print('two_stage', d['value'], [(round(s['kernel_ms_per_launch'],3), round(s['frac'],3)) for s in d['roofline_stages']])"

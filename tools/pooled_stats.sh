# pooled kernel (config5) pipeline counters and HIPER_DEBUG_MODE ablations
python __graft_entry__.py > gpurun_out/build.log 2>&1
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "hiper pipe" | tail -1
for M in 1 2 3; do
HIPER_DEBUG_MODE=$M timeout 300 python bench.py --workload config5 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('mode $M', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --workload config5 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('prod', d['value'], d['roofline']['achieved'], d['clocks']['sm_mhz'])"

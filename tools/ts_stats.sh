python __graft_entry__.py > gpurun_out/build.log 2>&1
for V in "" "HIPER_TS_N128=1"; do
env $V HIPER_MAXSIM_TS=1 HIPER_PIPE_STATS=1 timeout 300 python bench.py --chunks 300000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ts_stats.out 2> gpurun_out/ts_stats.err
echo "$V"; grep -i "pipe" gpurun_out/ts_stats.err | tail -1
env $V HIPER_MAXSIM_TS=1 timeout 300 python bench.py --chunks 300000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('TS $V', d['value'], d['roofline']['frac'])"
done
HIPER_MAXSIM_TS=1 HIPER_TS_N128=1 timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "topk_config1 or domain and topk or batch_inv" 2>&1 | tail -2

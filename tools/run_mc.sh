set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
HIPER_POOLED_MC=1 timeout 600 python -m pytest tests/test_gpu_pooled.py tests/test_gpu_rerank.py -q -x -p no:cacheprovider > gpurun_out/pytest_mc.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_mc.log
for MC in 0 1; do
HIPER_POOLED_MC=$MC timeout 300 python bench.py --workload config5 --no-cpu-baseline --no-e2e > gpurun_out/c5_mc$MC.json 2> gpurun_out/c5_mc$MC.err
HIPER_POOLED_MC=$MC HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/c5_mc${MC}_stats.err
done
echo all_done

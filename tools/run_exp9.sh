set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_packed.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_packed.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_packed.log
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config3v --fixed-len --chunks 200000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/mstats_fix.json 2> gpurun_out/mstats_fix.err
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config3v --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/mstats_c3v.json 2> gpurun_out/mstats_c3v.err
timeout 900 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/bench_c3v.json 2> gpurun_out/bench_c3v.err
timeout 300 python bench.py --workload config2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
echo all_done

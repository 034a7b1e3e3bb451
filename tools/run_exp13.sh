set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config3v --chunks 300000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2> gpurun_out/mstats_c3v.err
timeout 900 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/bench_c3v.json 2> gpurun_out/bench_c3v.err
timeout 600 python bench.py --workload config3v --fixed-len --chunks 300000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_fix.json 2> gpurun_out/b_fix.err
timeout 600 python bench.py --chunks 300000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_c3s.json 2> gpurun_out/b_c3s.err
echo all_done

set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config3v --chunks 300000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/mstats_c3v.json 2> gpurun_out/mstats_c3v.err
timeout 900 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/bench_c3v.json 2> gpurun_out/bench_c3v.err
timeout 300 python bench.py --workload config2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
B="python bench.py --workload config2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_c2.log 2>&1
echo all_done

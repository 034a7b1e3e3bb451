set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config3v --fixed-len --chunks 200000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/mstats_fix.json 2> gpurun_out/mstats_fix.err
HIPER_PIPE_STATS=1 timeout 300 python bench.py --chunks 200000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/mstats_c3.json 2> gpurun_out/mstats_c3.err
timeout 300 python bench.py --workload config3v --fixed-len --chunks 300000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_fix.json 2> gpurun_out/b_fix.err
timeout 300 python bench.py --chunks 300000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_c3s.json 2> gpurun_out/b_c3s.err
echo all_done

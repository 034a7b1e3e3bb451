# MODE 0 vs MODE 2 (argmax capture) on config2: pipeline wait counters and kernel times
python __graft_entry__.py > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config2 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "hiper pipe" | tail -2
HIPER_PIPE_STATS=1 timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e --steps 3 --warmup 3 2>&1 | grep "hiper pipe" | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:maxsim -s 6 -c 3 --csv --log-file gpurun_out/m0.csv python bench.py --workload config2 --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > /dev/null 2>&1
grep -o '"gpu__time_duration.sum","ns","[0-9]*"' gpurun_out/m0.csv | tail -3

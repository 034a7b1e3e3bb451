set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo rc=$? >> gpurun_out/bench_default.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
C="python bench.py --chunks 20000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $C > gpurun_out/plain3.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:maxsim -s 1 -c 1 -o gpurun_out/prof_maxsim $C > gpurun_out/ncu_full.log 2>&1
echo all_done

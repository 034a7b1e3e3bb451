# Round evidence: plain bench, launch list, DRAM traffic of the bench's own fused-kernel launch,
# and one ncu --set full capture (reduced corpus) of the fused kernel.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/plain_b.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --replay-mode application --clock-control none -k regex:maxsim -s 1 -c 1 --csv --log-file gpurun_out/traffic.csv $B > gpurun_out/ncu_traffic.log 2>&1
C="python bench.py --chunks 100000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $C > gpurun_out/plain_c.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:maxsim -s 1 -c 1 -o gpurun_out/prof_final $C > gpurun_out/ncu_full.log 2>&1
echo done

# Tensor-pipe activity of the MaxSim kernel in ablation modes 0 (production), 2 (no TMA, no
# epilogue), 3 (no TMA, full epilogue), config3 shape at 50k chunks.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config3 --chunks 50000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"
for v in 0 2 3; do
  HIPER_DEBUG_MODE=$v timeout 300 $B > gpurun_out/exp16_plain_$v.json 2>&1 && \
  HIPER_DEBUG_MODE=$v timeout 600 ncu --metrics $M --clock-control none -k regex:maxsim -s 1 -c 1 --csv $B > gpurun_out/exp16_ncu_$v.csv 2> gpurun_out/exp16_ncu_$v.err
done
echo all_done > gpurun_out/exp16_done

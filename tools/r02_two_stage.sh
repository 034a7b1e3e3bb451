# N3 two-stage workload: bench line, launch list, one full ncu capture of each stage's kernel.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload two_stage"
timeout 900 $B --steps 10 --warmup 3 > gpurun_out/ts_bench.json 2> gpurun_out/ts_bench.err
cat gpurun_out/ts_bench.json
S="$B --steps 2 --warmup 1 --no-cpu-baseline"
timeout 600 $S > gpurun_out/ts_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/ts_launches.csv $S > gpurun_out/ts_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rerank_gather -s 2 -c 1 \
  -o gpurun_out/ts_prof_rerank $S > gpurun_out/ts_ncu_rerank.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pooled_sm100 -s 2 -c 1 \
  -o gpurun_out/ts_prof_pooled $S > gpurun_out/ts_ncu_pooled.log 2>&1
ls -la gpurun_out/

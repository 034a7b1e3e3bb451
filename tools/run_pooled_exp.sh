# Pooled (a12) limiter experiment: per-SM throughput vs number of resident pairs; ncu of the full-size launch.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for P in 74 37 18; do HIPER_POOLED_PAIRS=$P timeout 600 $B > gpurun_out/pooled_p$P.json 2> gpurun_out/pooled_p$P.err; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pooled -s 3 -c 1 -o gpurun_out/prof_pooled_full python bench.py --workload config5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_pooled_full.log 2>&1
echo all_done

set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for D in 3 4; do HIPER_PIPE_STATS=1 HIPER_DEBUG_MODE=$D timeout 300 $B > gpurun_out/pstats$D.json 2> gpurun_out/pstats$D.err; done
C="python bench.py --workload config3v --chunks 100000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $C > gpurun_out/plain_pk.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:maxsim -s 1 -c 1 -o gpurun_out/prof_packed $C > gpurun_out/ncu_packed.log 2>&1
echo all_done

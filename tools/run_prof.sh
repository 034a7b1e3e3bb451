# usage: bash tools/run_prof.sh <tag> [extra bench args]  -- plain run then ncu --set full of one fused-kernel launch
TAG=$1; shift
C="python bench.py --chunks 20000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $*"
timeout 300 $C > gpurun_out/plain_$TAG.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:maxsim -s 1 -c 1 -o gpurun_out/prof_$TAG $C > gpurun_out/ncu_$TAG.log 2>&1
echo prof_rc=$?

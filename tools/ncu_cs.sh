set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
P="python bench.py --workload config5 --chunks 1200000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 300 $P > gpurun_out/plain_p.log 2>&1
for v in a32:HIPER_POOLED_CS_A=32 a64:HIPER_POOLED_CS_A=64 old:HIPER_POOLED_CS=0; do
  name=${v%%:*}; envs=${v#*:}
  env $envs timeout 900 ncu --set full --clock-control none --import-source on -k regex:pooled -s 1 -c 1 -o gpurun_out/prof_cs_$name $P > gpurun_out/ncu_cs_$name.log 2>&1
  python tools/ncu_summary.py gpurun_out/prof_cs_$name.ncu-rep 30 > gpurun_out/prof_cs_${name}_summary.txt 2>&1
  ncu -i gpurun_out/prof_cs_$name.ncu-rep --page raw --csv > gpurun_out/prof_cs_${name}_raw.csv 2>&1
  rm -f gpurun_out/prof_cs_$name.ncu-rep
done

# one ncu --set full capture of the MODE 2 (argmax) MaxSim kernel on config2 --grad
python __graft_entry__.py > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
B="python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:maxsim_sm100_pair -s 2 -c 1 -o gpurun_out/mode2 $B > gpurun_out/ncu_mode2.log 2>&1
tail -2 gpurun_out/ncu_mode2.log
ncu -i gpurun_out/mode2.ncu-rep --page details --csv > gpurun_out/mode2_details.csv 2>&1
ncu -i gpurun_out/mode2.ncu-rep --page source --csv --print-source sass > gpurun_out/mode2_source.csv 2>&1
ncu -i gpurun_out/mode2.ncu-rep --page raw --csv > gpurun_out/mode2_raw.csv 2>&1
rm -f gpurun_out/mode2.ncu-rep

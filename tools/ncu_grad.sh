# one ncu --set full capture of the N1 grad_d kernels (config2 --grad), summarised as csv
python __graft_entry__.py > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
B="python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"grad_d_seg" -s 1 -c 1 -o gpurun_out/grad_d $B > gpurun_out/ncu_grad.log 2>&1
tail -3 gpurun_out/ncu_grad.log
for k in grad_d_seg; do
ncu -i gpurun_out/grad_d.ncu-rep -k regex:$k --page details --csv > gpurun_out/${k}_details.csv 2>&1
ncu -i gpurun_out/grad_d.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/${k}_source.csv 2>&1
done
ls -la gpurun_out/

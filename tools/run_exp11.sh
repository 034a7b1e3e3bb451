set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
for MB in 24 12; do
HIPER_BAND_MB=$MB timeout 600 $B > gpurun_out/band_$MB.json 2> gpurun_out/band_$MB.err
HIPER_BAND_MB=$MB timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --replay-mode application --clock-control none -k regex:maxsim -s 1 -c 1 --csv --log-file gpurun_out/traffic_$MB.csv $B > gpurun_out/ncu_traffic_$MB.log 2>&1
done
echo all_done

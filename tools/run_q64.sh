set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --queries 64 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $B > gpurun_out/q64_base.json 2> gpurun_out/q64_base.err
HIPER_BAND_MB=0 timeout 300 $B > gpurun_out/q64_band0.json 2> gpurun_out/q64_band0.err
HIPER_LOCKSTEP_WINDOW=64 timeout 300 $B > gpurun_out/q64_w64.json 2> gpurun_out/q64_w64.err
HIPER_LOCKSTEP_WINDOW=32 timeout 300 $B > gpurun_out/q64_w32.json 2> gpurun_out/q64_w32.err
timeout 900 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --replay-mode application --clock-control none -k regex:maxsim -s 1 -c 1 --csv --log-file gpurun_out/traffic_q64.csv python bench.py --queries 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_q64.log 2>&1
echo all_done

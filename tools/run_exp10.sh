set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
HIPER_BAND_MB=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_noband.json 2> gpurun_out/bench_c3_noband.err
timeout 300 python bench.py --workload config2 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --replay-mode application --clock-control none -k regex:maxsim -s 1 -c 1 --csv --log-file gpurun_out/traffic.csv $B > gpurun_out/ncu_traffic.log 2>&1
echo all_done

set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_packed.py tests/test_gpu_pooled.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for MB in 0 48 24; do
HIPER_BAND_MB=$MB timeout 600 $B > gpurun_out/band_$MB.json 2> gpurun_out/band_$MB.err
done
for MB in 24; do
HIPER_BAND_MB=$MB timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --replay-mode application --clock-control none -k regex:maxsim -s 1 -c 1 --csv --log-file gpurun_out/traffic_$MB.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_traffic_$MB.log 2>&1
done
timeout 600 python bench.py --workload config5 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
echo all_done

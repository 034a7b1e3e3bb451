# Packed layout with replicated padding rows (no tail re-reads): parity, pipe stats, config3v/4v benches.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/pytest_packed.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_packed.log
HIPER_PIPE_STATS=1 timeout 600 python bench.py --workload config3v --chunks 300000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/pipe_c3v.json 2> gpurun_out/pipe_c3v.err
timeout 900 python bench.py --workload config3v --no-cpu-baseline > gpurun_out/bench_c3v.json 2> gpurun_out/bench_c3v.err
timeout 900 python bench.py --workload config4v --no-cpu-baseline > gpurun_out/bench_c4v.json 2> gpurun_out/bench_c4v.err
echo all_done

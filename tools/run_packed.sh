# N4 first GPU pass: packed-layout parity tests, then config3v bench packed vs dense.
set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_packed.py -q -x -p no:cacheprovider > gpurun_out/pytest_packed.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_packed.log
timeout 900 python bench.py --workload config3v --no-cpu-baseline > gpurun_out/bench_c3v.json 2> gpurun_out/bench_c3v.err; echo rc=$? >> gpurun_out/bench_c3v.err
timeout 900 python bench.py --workload config3v --no-pack --no-cpu-baseline --no-e2e > gpurun_out/bench_c3v_dense.json 2> gpurun_out/bench_c3v_dense.err; echo rc=$? >> gpurun_out/bench_c3v_dense.err
echo all_done

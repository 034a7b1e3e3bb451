set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1
B="python bench.py --workload config5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for D in 1 2; do HIPER_DEBUG_MODE=$D timeout 600 $B > gpurun_out/pooled_dbg$D.json 2> gpurun_out/pooled_dbg$D.err; done
timeout 900 python -m pytest tests/test_gpu_packed.py -q -x -p no:cacheprovider > gpurun_out/pytest_packed.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_packed.log
timeout 900 python bench.py --workload config3v --no-cpu-baseline --no-e2e > gpurun_out/bench_c3v.json 2> gpurun_out/bench_c3v.err
echo all_done

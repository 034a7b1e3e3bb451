# compute-sanitizer memcheck (one tool) on smoke(): the fused kernels, NORM layout, merge and loss.
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python __graft_entry__.py smoke > gpurun_out/memcheck_smoke.log 2>&1
echo rc=$? >> gpurun_out/memcheck_smoke.log

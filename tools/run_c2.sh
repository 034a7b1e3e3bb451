# ColTrast step (config2): forward and fwd+bwd bench lines (e2e with prefetched inputs).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python bench.py --workload config2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --workload config2 --grad > gpurun_out/bench_c2_grad.json 2> gpurun_out/bench_c2_grad.err
echo all_done >> gpurun_out/bench_c2.err

# Short N-GPU re-verification of the final tree: sharded == single check, multi-GPU tests, default bench, reference arm.
N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 $R --master-port 29511 tests/dist_topk_check.py > gpurun_out/dist_check_$N.log 2>&1; echo rc=$? >> gpurun_out/dist_check_$N.log
timeout 600 python -m pytest tests/test_multi_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi_$N.log
timeout 900 $R --master-port 29512 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 600 $R --master-port 29515 bench.py --gpus $N --impl reference > gpurun_out/bench_n${N}_ref.json 2> gpurun_out/bench_n${N}_ref.err
echo all_done

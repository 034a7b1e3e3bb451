N=${1:-2}
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tests/dist_topk_check.py > gpurun_out/dist_check_$N.log 2>&1; echo rc=$? >> gpurun_out/dist_check_$N.log
timeout 600 python -m pytest tests/test_multi_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --workload config4 > gpurun_out/bench_n${N}_c4.json 2> gpurun_out/bench_n${N}_c4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $N --workload config5 > gpurun_out/bench_n${N}_c5.json 2> gpurun_out/bench_n${N}_c5.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus $N --impl reference > gpurun_out/bench_n${N}_ref.json 2> gpurun_out/bench_n${N}_ref.err

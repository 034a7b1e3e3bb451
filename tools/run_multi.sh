N=${1:-2}
python __graft_entry__.py > gpurun_out/build.log 2>&1
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tests/dist_topk_check.py > gpurun_out/dist_check_$N.log 2>&1; echo rc=$? >> gpurun_out/dist_check_$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo rc=$? >> gpurun_out/bench_n$N.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --chunks 3600000 --k 100 --steps 3 --warmup 1 > gpurun_out/bench_n${N}_36m.json 2> gpurun_out/bench_n${N}_36m.err; echo rc=$? >> gpurun_out/bench_n${N}_36m.err

# N = 4, packed workloads only (after the packed pass-3 change): sharded == single check, config4v,
# and the paper-scale 16.4M-chunk semantic corpus.
N=${1:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 $R --master-port 29521 tests/dist_topk_check.py > gpurun_out/dist_check_$N.log 2>&1; echo rc=$? >> gpurun_out/dist_check_$N.log
timeout 1200 $R --master-port 29526 bench.py --gpus $N --workload config4v > gpurun_out/bench_n${N}_c4v.json 2> gpurun_out/bench_n${N}_c4v.err
timeout 1800 $R --master-port 29527 bench.py --gpus $N --workload config4v --chunks 16400000 --queries 256 --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_n4_c4v_16m.json 2> gpurun_out/bench_n4_c4v_16m.err
echo all_done

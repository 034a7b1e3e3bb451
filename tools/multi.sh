# Multi-GPU evidence at N = $1 (one box, N GPUs; run under gpurun --gpus N): the sharded top-k, N3 and
# N2 paths against the single-GPU result and the oracle (tests/dist_topk_check.py), then the strong-
# scaling bench lines.  $2 = "quick" runs the check and the default bench only.
N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 $R --master-port 29511 tests/dist_topk_check.py > gpurun_out/dist_check_$N.log 2>&1; echo rc=$? >> gpurun_out/dist_check_$N.log
timeout 900 $R --master-port 29512 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
if [ "$2" != "quick" ]; then
  timeout 1200 $R --master-port 29513 bench.py --gpus $N --workload config4 > gpurun_out/bench_n${N}_c4.json 2> gpurun_out/bench_n${N}_c4.err
  timeout 1200 $R --master-port 29516 bench.py --gpus $N --workload config4v > gpurun_out/bench_n${N}_c4v.json 2> gpurun_out/bench_n${N}_c4v.err
  timeout 900 $R --master-port 29514 bench.py --gpus $N --workload config5 > gpurun_out/bench_n${N}_c5.json 2> gpurun_out/bench_n${N}_c5.err
  timeout 900 $R --master-port 29517 bench.py --gpus $N --workload two_stage > gpurun_out/bench_n${N}_ts.json 2> gpurun_out/bench_n${N}_ts.err
  timeout 900 $R --master-port 29515 bench.py --gpus $N --impl reference > gpurun_out/bench_n${N}_ref.json 2> gpurun_out/bench_n${N}_ref.err
fi
tail -3 gpurun_out/dist_check_$N.log
echo all_done

# Multi-GPU evidence at N = $1 (one box, N GPUs): sharded == single (bitwise), strong scaling of the
# 1M corpus, the 3.6M corpus (dense config4 and semantic-packed config4v), pooled config5, the
# reference arm; at N = 4 also the paper-scale 16.4M-chunk semantic corpus.
N=${1:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 $R --master-port 29511 tests/dist_topk_check.py > gpurun_out/dist_check_$N.log 2>&1; echo rc=$? >> gpurun_out/dist_check_$N.log
timeout 600 python -m pytest tests/test_multi_gpu.py -q -p no:cacheprovider > gpurun_out/pytest_multi_$N.log 2>&1
timeout 900 $R --master-port 29512 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 1200 $R --master-port 29513 bench.py --gpus $N --workload config4 > gpurun_out/bench_n${N}_c4.json 2> gpurun_out/bench_n${N}_c4.err
timeout 1200 $R --master-port 29516 bench.py --gpus $N --workload config4v > gpurun_out/bench_n${N}_c4v.json 2> gpurun_out/bench_n${N}_c4v.err
timeout 900 $R --master-port 29514 bench.py --gpus $N --workload config5 > gpurun_out/bench_n${N}_c5.json 2> gpurun_out/bench_n${N}_c5.err
timeout 900 $R --master-port 29515 bench.py --gpus $N --impl reference > gpurun_out/bench_n${N}_ref.json 2> gpurun_out/bench_n${N}_ref.err
if [ "$N" = "4" ]; then
  timeout 1800 $R --master-port 29517 bench.py --gpus $N --workload config4v --chunks 16400000 --queries 256 --steps 2 --warmup 1 --no-e2e > gpurun_out/bench_n4_c4v_16m.json 2> gpurun_out/bench_n4_c4v_16m.err
fi
echo all_done

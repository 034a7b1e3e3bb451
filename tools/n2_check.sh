# N2 full loss: coltrast GPU tests, then peer-window vs NCCL gather at N = 2 (run under gpurun --gpus 2)
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -k "coltrast" -p no:cacheprovider > gpurun_out/pytest_n2.log 2>&1; tail -2 gpurun_out/pytest_n2.log
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 $R --master-port 29531 tests/dist_topk_check.py > gpurun_out/dist_check_2.log 2>&1; echo dist_rc=$?; grep -E "N=|DIST|ORACLE|oracle top" gpurun_out/dist_check_2.log | tail -9
for i in 1 2; do
timeout 600 $R --master-port 2953$((i+1)) bench.py --gpus 2 --workload config2 --full-loss --no-cpu-baseline > gpurun_out/n2_peer_$i.json 2> gpurun_out/n2_peer_$i.err
HIPER_N2_NCCL=1 timeout 600 $R --master-port 2954$i bench.py --gpus 2 --workload config2 --full-loss --no-cpu-baseline > gpurun_out/n2_nccl_$i.json 2> gpurun_out/n2_nccl_$i.err
done
for f in gpurun_out/n2_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us', d['extra'])" 2>&1 | tail -1; done

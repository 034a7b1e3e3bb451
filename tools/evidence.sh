# Round evidence on ONE GPU (run under gpurun from the repo root).  Stages, selectable as arguments
# (default: all): tests smoke bench ref workloads stats launches ncu.
#   tests      the GPU test suite                      -> gpurun_out/pytest_gpu.log
#   smoke      __graft_entry__.smoke()                 -> gpurun_out/smoke.log
#   bench      the default bench line (config3)        -> gpurun_out/bench_final.json
#   ref        bench.py --impl reference               -> gpurun_out/bench_ref.json
#   workloads  every other workload line               -> gpurun_out/bench_<workload>.json
#   stats      HIPER_PIPE_STATS counters               -> gpurun_out/pipe_stats.log
#   launches   ncu launch list + DRAM bytes of the fused kernel's bench launch
#   ncu        ncu --set full of each hot kernel       -> gpurun_out/prof_*.ncu-rep
set -x
STAGES=${*:-tests smoke bench ref workloads stats launches ncu}
has() { case " $STAGES " in *" $1 "*) return 0;; esac; return 1; }
python __graft_entry__.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if has tests; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
fi
if has smoke; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
fi
has bench && timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
has ref && timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if has workloads; then
  timeout 900 python bench.py --queries 64 --no-cpu-baseline > gpurun_out/bench_config3_q64.json 2> gpurun_out/bench_config3_q64.err
  for W in config3v config5 config2 two_stage; do
    timeout 900 python bench.py --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
  done
  timeout 900 python bench.py --workload config3v --no-pack --no-cpu-baseline > gpurun_out/bench_config3v_dense.json 2> gpurun_out/bench_config3v_dense.err
  timeout 900 python bench.py --workload config2 --grad --no-cpu-baseline > gpurun_out/bench_config2_grad.json 2> gpurun_out/bench_config2_grad.err
  timeout 1200 python bench.py --workload config4v --queries 256 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_config4v_n1.json 2> gpurun_out/bench_config4v_n1.err
fi
if has stats; then
  for W in "" "--workload config3v" "--workload config5"; do
    HIPER_PIPE_STATS=1 timeout 300 python bench.py $W --chunks 300000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>> gpurun_out/pipe_stats.log
  done
fi
if has launches; then
  B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 600 $B > gpurun_out/plain_b.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1 && \
    timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --replay-mode application --clock-control none -k regex:maxsim -s 1 -c 1 --csv --log-file gpurun_out/traffic.csv $B > gpurun_out/ncu_traffic.log 2>&1
fi
if has ncu; then
  C="python bench.py --chunks 100000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 300 $C > gpurun_out/plain_c.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:maxsim -s 1 -c 1 -o gpurun_out/prof_maxsim $C > gpurun_out/ncu_full.log 2>&1
  V="python bench.py --workload config3v --chunks 200000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 300 $V > gpurun_out/plain_v.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:maxsim -s 1 -c 1 -o gpurun_out/prof_packed $V > gpurun_out/ncu_packed.log 2>&1
  P="python bench.py --workload config5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 300 $P > gpurun_out/plain_p.log 2>&1 && \
    timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pooled -s 1 -c 1 -o gpurun_out/prof_pooled $P > gpurun_out/ncu_pooled.log 2>&1
fi
# keep gpurun_out under gpurun's 64 MiB copy-back limit: summarise the captures here, keep only the
# MaxSim report
for r in gpurun_out/prof_*.ncu-rep; do
  [ -f "$r" ] && python tools/ncu_summary.py "$r" 30 > "${r%.ncu-rep}_summary.txt" 2>&1
done
rm -f gpurun_out/prof_packed.ncu-rep gpurun_out/prof_pooled.ncu-rep
echo evidence_done

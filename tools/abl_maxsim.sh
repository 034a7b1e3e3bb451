# MaxSim pipeline ablations (lockstep, A buffers, window, band size): HIPER_PIPE_STATS counters per switch
python __graft_entry__.py > gpurun_out/build.log 2>&1
for V in "X=1" "HIPER_NO_LOCKSTEP=1" "HIPER_ONE_A=1" "HIPER_LOCKSTEP_WINDOW=64" "HIPER_BAND_MB=96"; do
  env $V HIPER_PIPE_STATS=1 timeout 300 python bench.py --chunks 300000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "hiper pipe" | tail -1 | sed "s/^/$V: /"
  env $V timeout 300 python bench.py --chunks 300000 --steps 4 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.load(sys.stdin); print('   ', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done

# A/B of grad_d segment sizes (HIPER_GRAD_S) on config2 --grad; launch list per setting
python __graft_entry__.py > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "grad" > gpurun_out/pytest_grad.log 2>&1; tail -1 gpurun_out/pytest_grad.log
for S in 128 256; do
  for i in 1 2; do
    HIPER_GRAD_S=$S timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S=$S', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us')"
  done
  HIPER_GRAD_S=$S timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:grad_d -s 12 -c 9 --csv --log-file gpurun_out/gab_$S.csv python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e --steps 3 --warmup 3 > /dev/null 2>&1
  python - <<P
import csv
rows=list(csv.reader(open('gpurun_out/gab_$S.csv')))
hdr=None; agg={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            k=d['Kernel Name'].split('(')[0][:40]; agg.setdefault(k,[]).append(float(d['Metric Value']))
for k,v in agg.items(): print(f"  S=$S {k:42s} {sum(v)/len(v)/1000:8.1f} us x{len(v)}")
P
done

# APPEND path: sample fraction A/B (HIPER_POOLED_SAMPLE_DIV) on the two-stage workload
python __graft_entry__.py > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
for D in 32; do
  for i in 1 2; do
    HIPER_POOLED_SAMPLE_DIV=$D timeout 600 python bench.py --workload two_stage --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('div=$D', round(d['value'],1), round(d['ms_per_step'],3), 'ms')"
  done
  HIPER_POOLED_SAMPLE_DIV=$D timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"pooled|cand_select|topk_merge" -s 8 -c 8 --csv --log-file gpurun_out/sab_$D.csv python bench.py --workload two_stage --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > /dev/null 2>&1
  python - <<P
import csv
rows=list(csv.reader(open('gpurun_out/sab_$D.csv')))
hdr=None; agg={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            k=d['Kernel Name'].split('(')[0][:46]; agg.setdefault(k,[]).append(float(d['Metric Value']))
for k,v in agg.items(): print(f"  div=$D {k:48s} {sum(v)/len(v)/1000:9.1f} us x{len(v)}")
P
done

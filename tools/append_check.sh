# pooled top-k APPEND path (k > 16): tests + two-stage bench A/B vs the heap path
python __graft_entry__.py > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "pooled or rerank or two_stage" > gpurun_out/pytest_append.log 2>&1; tail -3 gpurun_out/pytest_append.log
for i in 1 2; do
  timeout 600 python bench.py --workload two_stage --no-cpu-baseline 2>/dev/null > gpurun_out/ts_append_$i.json
  HIPER_POOLED_APPEND=0 timeout 600 python bench.py --workload two_stage --no-cpu-baseline 2>/dev/null > gpurun_out/ts_heap_$i.json
done
for f in gpurun_out/ts_*.json; do python -c "
import json; d=json.load(open('$f')); r=d.get('roofline') or {}
print('$f', round(d['value'],1), round(d['ms_per_step'],3), 'ms', [ (s.get('name'), round(s.get('frac',0),3)) for s in d.get('roofline_stages',[])] if d.get('roofline_stages') else r.get('frac'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"pooled|cand_select|topk_merge|rerank" -s 10 -c 12 --csv --log-file gpurun_out/ts_launches.csv python bench.py --workload two_stage --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > /dev/null 2>&1
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/ts_launches.csv')))
hdr=None; agg={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            k=d['Kernel Name'].split('(')[0][:50]; agg.setdefault(k,[]).append(float(d['Metric Value']))
for k,v in agg.items(): print(f"  {k:52s} {sum(v)/len(v)/1000:9.1f} us x{len(v)}")
P

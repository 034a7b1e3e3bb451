# N1 backward: grad/debug GPU tests, two config2 --grad bench lines, warm launch list of the step
python __graft_entry__.py > gpurun_out/build.log 2>&1 || tail -20 gpurun_out/build.log
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider -k "grad or debug" > gpurun_out/pytest_grad.log 2>&1; tail -3 gpurun_out/pytest_grad.log
for i in 1 2; do
timeout 300 python bench.py --workload config2 --grad --no-cpu-baseline > gpurun_out/grad_new_$i.json 2>/dev/null

done
for f in gpurun_out/grad_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step']*1000,1), 'us')"; done
B="python bench.py --workload config2 --grad --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 40 -c 30 --csv --log-file gpurun_out/grad_launches.csv $B > /dev/null 2>&1
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/grad_launches.csv')))
hdr=None; agg={}
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d.get('Metric Name')=='gpu__time_duration.sum':
            k=d['Kernel Name'].split('(')[0][:50]; agg.setdefault(k,[]).append(float(d['Metric Value']))
for k,v in agg.items(): print(f"{k:52s} {sum(v)/len(v)/1000:8.1f} us x{len(v)}")
P

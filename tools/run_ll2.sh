timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
MP_NO_LOOKAHEAD=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll2.csv python tools/probe_scaling.py 16384 --noprof > /dev/null 2>&1; echo ncu rc=$?
python3 - <<'PY'
import csv,re,collections
rows=list(csv.reader(open('gpurun_out/ll2.csv')))
hdr=None;data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
data=data[len(data)//2:]
agg=collections.defaultdict(list)
for d in data:
    name=re.sub(r"\(.*","",d["Kernel Name"]).replace("void ","").replace("unnamed>::","")
    agg[(name[:34],d['Grid Size'])].append(float(d['Metric Value'])/1e3)
for k,v in sorted(agg.items(), key=lambda x:-sum(x[1]))[:28]:
    print(f"{sum(v)/1e3:7.3f} ms n={len(v):4d} avg={sum(v)/len(v):7.1f}us  {k}")
PY

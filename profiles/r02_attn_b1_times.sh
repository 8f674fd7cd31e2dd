# per-launch device time of every attention launch in one batch-1 step (ncu, cold cache, serialised)
set -x
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k "regex:k_attn" --csv --log-file gpurun_out/attn_b1_times.csv python bench.py --profile-only --batch 1 --steps 1 --warmup 1 --no-baselines --no-cpu-baseline --pools random > /dev/null 2>&1; echo rc=$?
python - <<'PY'
import csv
lines=open('gpurun_out/attn_b1_times.csv').read().splitlines()
st=[i for i,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.reader(lines[st:])); h=rows[0]; rows=rows[1:]
ID,K,MN,MV=(h.index(x) for x in ("ID","Kernel Name","Metric Name","Metric Value"))
by={}
for r in rows:
    d=by.setdefault(r[ID],{"name":r[K][:40]}); d[r[MN]]=float(r[MV].replace(",",""))
ks=list(by.values())
print(len(ks),"launches; last 32:")
for x in ks[-32:]:
    print(x["name"], round(x["gpu__time_duration.sum"]/1e3,1), "us", round(x.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",0),1))
PY

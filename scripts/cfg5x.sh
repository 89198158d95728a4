timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cache1.csv python bench_cache.py --keys 1000000 --capacity 100000 --reps 3 --max-batch 1 --warmup-mult 0.001 --no-cpu --eager > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=list(csv.reader(open('gpurun_out/launches_cache1.csv')))
hdr=None;seq=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r;continue
    if hdr and len(r)==len(hdr):
        try: seq.append((r[hdr.index('Kernel Name')][:70], float(r[hdr.index('Metric Value')].replace(',',''))/1000))
        except: pass
# last ~40 launches = the last lookups
for k,v in seq[-45:]: print(f"{v:8.2f} {k}")
PY

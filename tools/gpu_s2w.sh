timeout 600 python -m pytest tests/test_gpu_qr_blocked.py -x -q 2>&1 | tail -2
for lv in 32 64; do timeout 120 python tools/qr_probe.py 6144 2048 $lv; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2w_launch64.csv python tools/qr_probe.py 6144 2048 64 > /dev/null 2>&1
python - <<'P'
import csv, collections
rows=list(csv.reader(open('gpurun_out/s2w_launch64.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
hdr=rows[hi]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Value')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[hi+1:]:
    try: v=float(r[mi].replace(',',''))/1e6
    except: continue
    agg[r[ki].split('(')[0][:60]][0]+=1; agg[r[ki].split('(')[0][:60]][1]+=v
for k,(c,ms) in sorted(agg.items(), key=lambda x:-x[1][1])[:12]: print(f'{k:60s}{c:6d} {ms:9.2f} ms')
P

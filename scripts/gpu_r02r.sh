mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:hop_kernel -c 20 --csv --log-file gpurun_out/launches_C5_lat.csv python bench.py --hops 64 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 30 > gpurun_out/ncu_lat.log 2>&1; echo "rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches_C5_lat.csv')))
hdr=None
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        print(d['Kernel Name'][:50], d['Metric Name'], d['Metric Value'])
PY

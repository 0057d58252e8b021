# session 6: one-hop kernel with an early bulk L2 prefetch of each partition group's first rows (tuning hop_pf), latency leg
B="python bench.py --hops 128 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for t in "C3 hop_pf=0" "C3 hop_pf=8" "C3 hop_pf=16" "C3 hop_pf=32" "C3 hop_pf=64" "C3 hop_pf=0" "C3 hop_pf=16" "C4 hop_pf=0" "C4 hop_pf=8" "C4 hop_pf=32" "C5 hop_pf=0" "C5 hop_pf=16" "C5 hop_pf=64" "C2 hop_pf=0" "C2 hop_pf=16"; do
  set -- $t
  timeout 300 $B --config $1 --tune $2 > gpurun_out/s6f.json 2> gpurun_out/s6f.err
  python -c "
import json
d=json.load(open('gpurun_out/s6f.json'))['latency']
print('$t', 'gpu p50 %.4f p99 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['kernel_roofline']['kernel_us_live']))
"
done

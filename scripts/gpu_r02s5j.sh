# session 5: one-hop kernel geometry (CTAs per source) for the bank configs, latency leg
B="python bench.py --hops 128 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for c in C3 C5; do
for t in "p=1" "p=2" "p=4" "p=1 nt=512" "p=2 nt=512" "p=1"; do
  a=""; for kv in $t; do a="$a --tune $kv"; done
  $B --config $c $a > gpurun_out/s5j.json 2> gpurun_out/s5j.err
  python -c "
import json
d=json.load(open('gpurun_out/s5j.json'))['latency']
print('$c $t', 'gpu p50 %.4f p99 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['kernel_roofline']['kernel_us_live']))
"
done; done

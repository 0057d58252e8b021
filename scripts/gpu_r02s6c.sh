# session 6: one-hop kernel threads per CTA, second pass (C5 small CTAs, C3 nt=512 now that nt drives the launch)
B="python bench.py --hops 128 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for t in "C5 nt=0" "C5 nt=64" "C5 nt=32" "C5 nt=0" "C5 nt=64" "C5 nt=32" "C3 nt=512" "C3 nt=0" "C4 nt=0" "C4 nt=512" "C4 nt=1024" "C2 nt=0" "C2 nt=512" "C2 nt=128"; do
  set -- $t
  timeout 300 $B --config $1 --tune $2 > gpurun_out/s6c.json 2> gpurun_out/s6c.err
  python -c "
import json
d=json.load(open('gpurun_out/s6c.json'))['latency']
print('$t', 'gpu p50 %.4f p99 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['kernel_roofline']['kernel_us_live']))
"
done

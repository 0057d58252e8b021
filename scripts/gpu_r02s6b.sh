# session 6: one-hop kernel threads per CTA on C3 (1024 CTAs: 256 threads -> 4 resident / SM = 1.73 waves;
# 128 threads -> 7 resident / SM by shared memory = one wave), latency leg, in-place pinned calls
B="python bench.py --hops 128 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for c in C3 C5; do
for t in "nt=0" "nt=128" "nt=64" "nt=0" "nt=128"; do
  a=""; for kv in $t; do a="$a --tune $kv"; done
  timeout 300 $B --config $c $a > gpurun_out/s6b.json 2> gpurun_out/s6b.err
  python -c "
import json
d=json.load(open('gpurun_out/s6b.json'))['latency']
print('$c $t', 'gpu p50 %.4f p99 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['kernel_roofline']['kernel_us_live']))
"
done; done
timeout 300 python -m pytest tests/test_gpu_engine.py -x -q -k "launch or geometry or config" 2>&1 | tail -3

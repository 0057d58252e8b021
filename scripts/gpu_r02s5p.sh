# session 5: complex MACs on packed FP32 FMAs (FFMA2, fma.rn.f32x2) — same roundings, half the FMA issue slots
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/s5p_gputest.txt
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
for c in C5 C3 C2 C4 C1; do
  $B --config $c > gpurun_out/s5p_$c.json 2> gpurun_out/s5p_$c.err
  python -c "
import json
d=json.load(open('gpurun_out/s5p_$c.json'))
l=d.get('latency') or {}
print('$c', '%.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], d['roofline']['bound'], '%.3f'%d['roofline']['frac'], 'p50', l.get('gpu_ms_p50'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
"
done

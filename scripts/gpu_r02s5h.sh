# session 5: one-hop process() on pinned buffers in place (zero_copy) vs the copying path: latency leg
python -m pytest tests/test_gpu_edge.py tests/test_gpu_engine.py -x -q 2>&1 | tail -3
B="python bench.py --hops 128 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for c in C5 C3 C4 C2 C1; do
for k in 0 1 0 1; do
  $B --config $c --tune zero_copy=$k > gpurun_out/s5h_${c}_$k.json 2> gpurun_out/s5h_${c}_$k.err
  python -c "
import json
d=json.load(open('gpurun_out/s5h_${c}_$k.json'))['latency']
print('$c zero_copy=$k', 'gpu p50 %.4f p99 %.4f host p50 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['host_ms_p50'], d['kernel_roofline']['kernel_us_live']))
"
done; done

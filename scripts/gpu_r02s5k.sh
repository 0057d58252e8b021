# session 5: persistent bulk-copy ring kernel for one-hop calls of bank engines: parity, then latency A/B over ring geometries
timeout 600 python -m pytest tests/test_gpu_engine.py -x -q -k "ring" 2>&1 | tail -5
B="timeout 300 python bench.py --hops 128 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for c in C5 C3; do
for k in 0 1 2 3 4 0; do
  $B --config $c --tune hop_ring=$k > gpurun_out/s5k_${c}_$k.json 2> gpurun_out/s5k_${c}_$k.err
  python -c "
import json
d=json.load(open('gpurun_out/s5k_${c}_$k.json'))['latency']
print('$c hop_ring=$k', 'gpu p50 %.4f p99 %.4f host p50 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['host_ms_p50'], d['kernel_roofline']['kernel_us_live']))
"
done; done

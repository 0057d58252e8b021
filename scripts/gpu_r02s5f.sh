# session 5: one-hop kernel of bank engines with an L2 residency policy (bank rows partly evict-last, delay line evict-first)
python -m pytest tests/test_gpu_engine.py tests/test_gpu_edge.py -x -q 2>&1 | tail -3
B="python bench.py --hops 128 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for c in C5 C3; do
for k in 0 1 2 3 4 0; do
  $B --config $c --tune hop_l2_keep=$k > gpurun_out/s5f_${c}_$k.json 2> gpurun_out/s5f_${c}_$k.err
  python -c "
import json
d=json.load(open('gpurun_out/s5f_${c}_$k.json'))['latency']
print('$c keep=$k', 'p50 %.4f p99 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['kernel_roofline']['kernel_us_live']))
"
done; done

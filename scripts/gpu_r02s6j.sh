# session 6: why is the C3 one-hop kernel 98-105 us inside bench.py's latency leg but 67-73 us in scripts/hop_waves.py?
B="python bench.py --config C3 --steps 1 --warmup 3 --no-cpu --no-e2e --latency-hops 400"
for t in "--hops 128" "--hops 8" "--hops 128 --tune zero_copy=0" "--hops 8 --tune zero_copy=0"; do
  timeout 300 $B $t > gpurun_out/s6j.json 2> gpurun_out/s6j.err
  python -c "
import json
d=json.load(open('gpurun_out/s6j.json'))['latency']
print('$t', 'gpu p50 %.4f p99 %.4f kernel_us %.1f'%(d['gpu_ms_p50'], d['gpu_ms_p99'], d['kernel_roofline']['kernel_us_live']))
"
done
timeout 300 python scripts/hop_waves.py 2>&1 | tail -4

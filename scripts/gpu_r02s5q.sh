# session 5: bank pass memory budget (hops per pass): fewer Xe history copies / pass boundaries
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
for c in C5 C3; do
for t in "bank_pass_mb=32768" "bank_pass_mb=65536" "bank_pass_mb=98304" "bank_pass_mb=32768"; do
  $B --config $c --tune $t > gpurun_out/s5q.json 2> gpurun_out/s5q.err
  python -c "
import json
d=json.load(open('gpurun_out/s5q.json'))
print('$c $t', '%.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], d['path'], d['clocks']['sm_mhz'])
"
done; done

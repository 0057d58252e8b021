# session 5: C3 e2e with 16- vs 32-hop bank tiles
B="python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --latency-hops 0"
for t in "bank_pass_jh=8" "bank_pass_jh=16" "bank_pass_jh=8" "bank_pass_jh=16"; do
  $B --tune $t > gpurun_out/s5t.json 2> gpurun_out/s5t.err
  python -c "
import json
d=json.load(open('gpurun_out/s5t.json'))
print('C3 $t', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ms %.2f'%d['ms_per_step'], 'e2e ms %.2f'%d['e2e']['ms_per_step'], d['clocks']['sm_mhz'])
"
done

# session 5: partition groups Q again on the final bank MAC
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
for t in "C5 bank_pass_q=7" "C5 bank_pass_q=8" "C5 bank_pass_q=9" "C5 bank_pass_q=7" "C3 bank_pass_q=4" "C3 bank_pass_q=5" "C3 bank_pass_q=3" "C3 bank_pass_q=4"; do
  set -- $t
  $B --config $1 --tune $2 > gpurun_out/s5u.json 2> gpurun_out/s5u.err
  python -c "
import json
d=json.load(open('gpurun_out/s5u.json'))
print('$t', '%.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], d['clocks']['sm_mhz'])
"
done

# session 5: bank MAC groups accumulating in place (flags + tickets) vs Q partials summed by K5
timeout 300 python -m pytest tests/test_gpu_bank_pass.py -x -q 2>&1 | tail -5
B="timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
for t in "C5 bank_pass_inplace=0" "C5 bank_pass_inplace=1" "C5 bank_pass_inplace=0" "C5 bank_pass_inplace=1" "C3 bank_pass_inplace=0" "C3 bank_pass_inplace=1" "C3 bank_pass_inplace=0" "C3 bank_pass_inplace=1"; do
  set -- $t
  $B --config $1 --tune $2 > gpurun_out/s5v.json 2> gpurun_out/s5v.err
  python -c "
import json
d=json.load(open('gpurun_out/s5v.json'))
print('$t', '%.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], d['path'], d['clocks']['sm_mhz'])
"
done

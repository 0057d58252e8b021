mkdir -p gpurun_out
for q in 4 5 6 7; do
  timeout 600 python bench.py --steps 3 --warmup 3 --latency-hops 0 --no-cpu --no-e2e --tune bank_pass_q=$q > gpurun_out/q_$q.json 2> gpurun_out/q_$q.err
  python -c "
import json;d=json.load(open('gpurun_out/q_$q.json'));r=d['roofline'];print('Q=$q %.4g'%d['value'], 'ms/step %.1f'%d['ms_per_step'], 'mac %.2f'%r['avg_launch_ms'], 'share %.3f'%r['kernel_share_of_step'], d['clocks']['sm_mhz'])"
done

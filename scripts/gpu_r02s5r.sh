# session 5: 32-hop tiles (JH = 16, 512 threads, one CTA per SM) for the two-ear bank MAC (C3)
python -m pytest tests/test_gpu_bank_pass.py -x -q 2>&1 | tail -3
B="python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
for t in "bank_pass_jh=8" "bank_pass_jh=16" "bank_pass_jh=8" "bank_pass_jh=16"; do
  $B --tune $t > gpurun_out/s5r.json 2> gpurun_out/s5r.err
  python -c "
import json
d=json.load(open('gpurun_out/s5r.json'))
print('C3 $t', '%.4g'%d['value'], 'ms %.2f'%d['ms_per_step'], '%.2f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])
"
done

# session 5: bank MAC without loads past the partition group, idle warps of short tiles skipped, full tiles + remainder
python -m pytest tests/test_gpu_bank_pass.py tests/test_gpu_configs.py tests/test_gpu_multi_rank.py -x -q 2>&1 | tail -3 > gpurun_out/s5d_tests.txt; cat gpurun_out/s5d_tests.txt
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
for i in 1 2; do
for c in C5 C3; do
  $B --config $c > gpurun_out/s5d_${c}_$i.json 2> gpurun_out/s5d_${c}_$i.err
  python -c "
import json
d=json.load(open('gpurun_out/s5d_${c}_$i.json'))
print('$c', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], '%.2f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['roofline']['frac'])
"
done; done

# session 5: bank MAC tiles per CTA (L1 reuse of the Xe window) x tile size, C5 and C3
python -m pytest tests/test_gpu_bank_pass.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3 > gpurun_out/s5b_tests.txt
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
i=0
for t in "bank_pass_tpc=1" "bank_pass_tpc=0" "bank_pass_tpc=1 bank_pass_jh=32" "bank_pass_tpc=0 bank_pass_jh=32" "bank_pass_tpc=4 bank_pass_jh=32" "bank_pass_tpc=0 bank_pass_jh=32 bank_pass_q=6" "bank_pass_tpc=0 bank_pass_jh=8"; do
  i=$((i+1)); a=""; for kv in $t; do a="$a --tune $kv"; done
  $B $a > gpurun_out/s5b_c5_$i.json 2> gpurun_out/s5b_c5_$i.err
  python -c "
import json
d=json.load(open('gpurun_out/s5b_c5_$i.json'))
print('C5', '$t', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], '%.2f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])
"
done
for t in "bank_pass_tpc=1" "bank_pass_tpc=0" "bank_pass_tpc=4"; do
  i=$((i+1)); a=""; for kv in $t; do a="$a --tune $kv"; done
  $B --config C3 $a > gpurun_out/s5b_c3_$i.json 2> gpurun_out/s5b_c3_$i.err
  python -c "
import json
d=json.load(open('gpurun_out/s5b_c3_$i.json'))
print('C3', '$t', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], '%.2f'%d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])
"
done
cat gpurun_out/s5b_tests.txt

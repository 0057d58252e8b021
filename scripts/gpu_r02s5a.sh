# session 5: 64-point K1 with 8 lanes per frame, parallel K5 overlap-add, JH = 32 bank tiles (C5)
python -m pytest tests/test_gpu_bank_pass.py tests/test_gpu_configs.py tests/test_gpu_wide.py -x -q 2>&1 | tail -5 > gpurun_out/s5a_tests.txt
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --latency-hops 0"
$B --tune k1_small=0 > gpurun_out/s5a_k1old.json 2> gpurun_out/s5a_k1old.err
$B > gpurun_out/s5a_new.json 2> gpurun_out/s5a_new.err
$B --tune bank_pass_jh=32 > gpurun_out/s5a_jh32.json 2> gpurun_out/s5a_jh32.err
$B --tune bank_pass_jh=32 --tune bank_pass_q=6 > gpurun_out/s5a_jh32q6.json 2> gpurun_out/s5a_jh32q6.err
$B > gpurun_out/s5a_new2.json 2> gpurun_out/s5a_new2.err
cat gpurun_out/s5a_tests.txt
for f in k1old new jh32 jh32q6 new2; do python -c "
import json,sys
d=json.load(open('gpurun_out/s5a_$f.json'))
print('$f', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['kernel_share_of_step'], d['clocks']['sm_mhz'])
"; done

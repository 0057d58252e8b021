mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bank_pass.py tests/test_gpu_configs.py tests/test_gpu_multi_rank.py -x -q > gpurun_out/bank_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bank_test.log
tail -2 gpurun_out/bank_test.log
for c in C5 C3; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --latency-hops 0 > gpurun_out/bq_$c.json 2> gpurun_out/bq_$c.err
python -c "
import json;d=json.load(open('gpurun_out/bq_$c.json'));r=d['roofline'];print('$c %.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ms/step %.1f'%d['ms_per_step'], 'par', d['parity']['rel_err_vs_reference'], d['clocks']['sm_mhz'])"
done

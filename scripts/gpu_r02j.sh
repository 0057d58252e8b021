mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_period.py tests/test_gpu_wide.py -x -q > gpurun_out/period_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/period_test.log
tail -4 gpurun_out/period_test.log
for t in 1 0; do
timeout 900 python bench.py --config C2 --steps 5 --warmup 3 --latency-hops 0 --no-cpu --no-e2e --tune wide_period=$t > gpurun_out/bench_C2_p$t.json 2> gpurun_out/bench_C2_p$t.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_C2_p$t.json'));r=d['roofline'];print('C2 wide_period=$t %.4g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'avg launch %.3f ms'%r['avg_launch_ms'], r['launches'], d['clocks']['sm_mhz'])"
done

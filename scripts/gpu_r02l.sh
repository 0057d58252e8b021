mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_wide.py tests/test_gpu_period.py tests/test_gpu_configs.py -x -q > gpurun_out/wide_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/wide_test.log
tail -3 gpurun_out/wide_test.log
for c in C2 C1; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --latency-hops 0 --no-cpu --no-e2e > gpurun_out/bench_${c}_kpf.json 2> gpurun_out/bench_${c}_kpf.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_${c}_kpf.json'));r=d['roofline'];print('$c %.4g'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'avg launch %.3f ms'%r['avg_launch_ms'], r['launches'], d['clocks'])"
done

mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_period.py -x -q > gpurun_out/period_test.log 2>&1; echo "pytest rc=$?" >> gpurun_out/period_test.log
tail -4 gpurun_out/period_test.log
timeout 900 python bench.py --config C4 --steps 3 --warmup 3 --latency-hops 0 --no-cpu --no-e2e > gpurun_out/bench_C4_period9.json 2> gpurun_out/bench_C4_period9.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/bench_C4_period9.json'));r=d['roofline'];print('C4 %.3g'%d['value'], 'avg launch %.2f ms'%r['avg_launch_ms'], r['launches'], d['clocks'])"

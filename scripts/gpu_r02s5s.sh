# session 5: ncu of the C3 bank MAC with 32-hop tiles, then the C3 line and the bank pass tests on the new default
python -m pytest tests/test_gpu_bank_pass.py tests/test_gpu_configs.py tests/test_gpu_multi_rank.py tests/test_gpu_bench_launch.py -x -q 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bank_mac -c 1 -o gpurun_out/s5s_ncu_C3_bank python bench.py --config C3 --hops 1024 --steps 1 --warmup 1 --no-cpu --no-e2e --latency-hops 0 > gpurun_out/s5s_ncu_C3_bank.log 2>&1; echo "ncu C3 rc=$?"
python bench.py --config C3 > gpurun_out/s5s_bench_C3.json 2> gpurun_out/s5s_bench_C3.err; echo "C3 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/s5s_bench_C3.json'))
l=d.get('latency') or {}
print('C3', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ms %.2f'%d['ms_per_step'], d['roofline']['bound'], '%.3f'%d['roofline']['frac'], 'p50', l.get('gpu_ms_p50'), 'par', d['parity']['rel_err_vs_reference'], d['clocks']['sm_mhz'])
"

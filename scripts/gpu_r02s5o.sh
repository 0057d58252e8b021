# session 5: bench lines of the other configs on the final tree
for c in C3 C2 C4 C1; do python bench.py --config $c > gpurun_out/s5o_bench_$c.json 2> gpurun_out/s5o_bench_$c.err; echo "$c rc=$?"; done
for c in C3 C2 C4 C1; do python -c "
import json
d=json.load(open('gpurun_out/s5o_bench_$c.json'))
l=d.get('latency') or {}
print('$c', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ms %.2f'%d['ms_per_step'], d['roofline']['bound'], '%.3f'%d['roofline']['frac'], 'p50', l.get('gpu_ms_p50'), 'cpu %.3g'%d['cpu_baseline']['value'], 'par', d['parity']['rel_err_vs_reference'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
"; done

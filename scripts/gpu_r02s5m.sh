# session 5 (after the ring-kernel opt-in): full GPU suite + smoke + default bench + reference arm on the final tree
python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/s5m_gputest.txt; cat gpurun_out/s5m_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5m_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --impl reference > gpurun_out/s5m_bench_ref.json 2> gpurun_out/s5m_bench_ref.err; echo "ref rc=$?"
python bench.py > gpurun_out/s5m_bench_C5.json 2> gpurun_out/s5m_bench_C5.err; echo "C5 rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/s5m_bench_C5.json'))
l=d['latency']
print('C5', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ms %.2f'%d['ms_per_step'], d['roofline']['bound'], '%.3f'%d['roofline']['frac'], 'p50', l['gpu_ms_p50'], l['gpu_ms_p99'], 'cpu %.3g'%d['cpu_baseline']['value'], 'par', d['parity'], d['clocks'])
"

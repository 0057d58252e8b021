# session 6: GPU tests + C5 default bench after the 64-thread rule for the one-hop kernel on C5-like bank engines
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/s6d_gputest.txt; cat gpurun_out/s6d_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6d_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/s6d_C5.json 2> gpurun_out/s6d_C5.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads(open("gpurun_out/s6d_C5.json").read().strip().splitlines()[-1])
l=d["latency"]
print("%.4g"%d["value"], "e2e %.4g"%d["e2e"]["value"], d["clocks"]["sm_mhz"], d["roofline"]["frac"], l["gpu_ms_p50"], l["gpu_ms_p99"], l["kernel_roofline"]["kernel_us_live"], l["kernel_roofline"]["frac"], d["parity"]["ok"])
PY

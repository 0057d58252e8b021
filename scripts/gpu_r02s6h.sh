# session 6: the other BASELINE configs on the final tree (one bench line each)
for c in C3 C4 C2 C1; do
  timeout 900 python bench.py --config $c > gpurun_out/s6h_$c.json 2> gpurun_out/s6h_$c.err; echo $c rc=$?
  python - <<PY
import json
d=json.loads(open("gpurun_out/s6h_$c.json").read().strip().splitlines()[-1])
l=d.get("latency") or {}
print("$c", "%.4g"%d["value"], "e2e %.4g"%d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["roofline"]["bound"], "%.3f"%d["roofline"]["frac"], l.get("gpu_ms_p50"), (d.get("parity") or {}).get("ok"))
PY
done

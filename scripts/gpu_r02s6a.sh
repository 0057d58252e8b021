# session 6: evidence on HEAD after the container was re-created (fresh build of every .so)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/s6a_gputest.txt; cat gpurun_out/s6a_gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6a_smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/s6a_smoke.log
timeout 600 python bench.py --impl reference > gpurun_out/s6a_ref.json 2> gpurun_out/s6a_ref.err; echo ref rc=$?
timeout 900 python bench.py > gpurun_out/s6a_C5.json 2> gpurun_out/s6a_C5.err; echo bench rc=$?
python - <<'PY'
import json
for f in ("s6a_ref","s6a_C5"):
    d=json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, "%.4g"%d["value"], "e2e %.4g"%d["e2e"]["value"], d.get("clocks",{}).get("sm_mhz"), d.get("roofline",{}).get("frac"), (d.get("latency") or {}).get("gpu_ms_p50"), d.get("parity"))
PY

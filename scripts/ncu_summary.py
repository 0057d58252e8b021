"""Summarise an `ncu --set full` capture (.ncu-rep) into profiles/ncu_summary_<config>.json:
per-launch duration, DRAM bytes and L2<->SM bytes, and their per-hop values (`per_hop`: the
bytes bench.py's roofline sides divide by the live launch time), plus the headline throughput /
occupancy / stall counters. Reads the report with `ncu -i --page raw`. `--kernel-match` picks the
launch the per-hop figures come from (default: the first)."""
import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "msecond": 1e3, "usecond": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3, "%": 1.0, "": 1.0}
KEEP = ["gpu__time_duration.sum", "lts__t_sectors.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar_write_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--config", required=True)
    ap.add_argument("--kernel", required=True, help="description of the captured kernel / geometry")
    ap.add_argument("--source", required=True, help="the command the capture ran")
    ap.add_argument("--alg-bytes", type=float, default=None, help="SURVEY 8(d) algorithmic bytes per launch")
    ap.add_argument("--hops-per-launch", type=float, default=None,
                    help="hops one captured launch processes (bench.py scales traffic per hop by its own launches)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--kernel-match", default=None, help="substring of the launch the per-hop figures come from")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    launches = []
    for r in data:
        d = {"name": r[hdr.index("Kernel Name")]}
        for k in KEEP:
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
                except ValueError:
                    d[k] = r[i]
        pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
        stalls = {h[len(pre):-len(suf)]: float(r[i].replace(",", "")) for i, h in enumerate(hdr)
                  if h.startswith(pre) and h.endswith(suf) and r[i] not in ("", "n/a")}
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        launches.append(d)
    sel = [l for l in launches if a.kernel_match is None or a.kernel_match in l["name"]] or launches
    n = len(sel)
    mean = lambda k: sum(l.get(k, 0.0) or 0.0 for l in sel) / n  # noqa: E731
    hpl = a.hops_per_launch
    per_hop = None
    if hpl:
        per_hop = {"dram_bytes": (mean("dram__bytes_read.sum") + mean("dram__bytes_write.sum")) / hpl,
                   "l2_read_bytes": mean("l1tex__m_xbar2l1tex_read_bytes.sum") / hpl,
                   "l2_write_bytes": mean("l1tex__m_l1tex2xbar_write_bytes.sum") / hpl,
                   "lts_bytes": 32 * mean("lts__t_sectors.sum") / hpl,
                   "duration_us": mean("gpu__time_duration.sum") / hpl}
    rd, wr = mean("dram__bytes_read.sum"), mean("dram__bytes_write.sum")
    out = {"kernel": a.kernel, "source": a.source, "launches_captured": n,
           "duration_us_cold": mean("gpu__time_duration.sum"),
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "l2_bytes_per_launch": 32 * mean("lts__t_sectors.sum") if "lts__t_sectors.sum" in hdr else None,
           "algorithmic_bytes_per_launch_8d": a.alg_bytes,
           "hops_per_launch": a.hops_per_launch,
           "dram_bytes_per_hop": (rd + wr) / a.hops_per_launch if a.hops_per_launch else None,
           "per_hop": per_hop,
           "lts_throughput_pct": mean("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
           "dram_throughput_pct": mean("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
           "l2_hit_pct": mean("lts__t_sector_hit_rate.pct"),
           "top_stalls": sel[0].get("top_stalls"),
           "note": "ncu flushes caches before each replay (cold); in the timed bench the C1/C2 delay line and "
                   "filter pool are L2-resident",
           "per_launch": launches}
    path = Path(a.out) if a.out else ROOT / "profiles" / f"ncu_summary_{a.config}.json"
    path.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: v for k, v in out.items() if k != "per_launch"}, indent=1))


if __name__ == "__main__":
    main()

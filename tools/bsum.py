"""Summarise bench.py JSON lines (one per file): value, e2e, stage ms."""
import json
import sys

for p in sys.argv[1:]:
    try:
        ln = [l for l in open(p) if l.startswith("{")][-1]
    except (IndexError, OSError):
        print(p, "no json")
        continue
    d = json.loads(ln)
    if "impl" in d:
        print(p, "REF", round(d["value"], 3), d["cpu_baseline"].get("rsvd_1thread"), d["cpu_baseline"]["cores"])
        continue
    pl = d.get("pipeline", {})
    st = {k: round(v, 3) for k, v in pl.get("stage_ms_per_step", {}).items()}
    print(p, d["config"]["workload"], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 3),
          "e2e", round(d["e2e"]["value"], 1), "roof", d.get("roofline", {}).get("frac"),
          "clk", (d.get("clocks") or {}).get("sm_mhz"))
    print("   ", st, "sweeps", pl.get("jacobi_sweeps"), "tsvd", (d.get("gpu_tsvd") or {}).get("value"))

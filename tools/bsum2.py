"""Print the headline fields of bench JSON lines: python tools/bsum2.py gpurun_out/x/bench_*.json"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "ERR", e)
        continue
    r = d.get("roofline") or {}
    print(f.split("/")[-1], round(d.get("value", 0), 2), "ms", round(d.get("ms_per_step", 0), 3), "e2e",
          round((d.get("e2e") or {}).get("value") or 0, 1), "roof", r.get("achieved") and round(r["achieved"], 1),
          r.get("unit"), r.get("frac") and round(r["frac"], 3), d.get("clocks"))
    if "pipeline" in d:
        print("   ", {k: round(v, 3) for k, v in d["pipeline"].get("stage_ms_per_step", {}).items()})

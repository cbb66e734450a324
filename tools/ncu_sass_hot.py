"""Hot SASS regions of one kernel in an ncu report: warp-stall samples per
instruction, with the surrounding instructions for context.

  python tools/ncu_sass_hot.py gpurun_out/prof.ncu-rep [top] [bins]
"""
import csv
import io
import subprocess
import sys


def main(path, top=20, bins=20):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    vals = []
    for r in rows[2:]:
        try:
            vals.append((float(r[si]), r[src].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(v for v, _ in vals) or 1.0
    n = len(vals)
    print(f"# {n} SASS instructions; sample share per {n // bins}-instruction bin:")
    for b in range(bins):
        a, e = b * n // bins, (b + 1) * n // bins
        ops = {}
        for _, s in vals[a:e]:
            op = s.split()[0] if s else ""
            if op.startswith("@"):
                op = s.split()[1]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + 1
        key = ",".join(k for k, _ in sorted(ops.items(), key=lambda x: -x[1])[:5])
        print(f"  [{a:5d},{e:5d}) {100 * sum(v for v, _ in vals[a:e]) / tot:5.1f}%  {key}")
    print("# top instructions")
    for v, i, s in sorted(((v, i, s) for i, (v, s) in enumerate(vals)), reverse=True)[:top]:
        print(f"  {100 * v / tot:5.1f}% [{i}] {s[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:]))

"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total device time and share.  Usage:
    python tools/ncu_launch_shares.py gpurun_out/launches.csv [first_n_launches]"""
import collections
import csv
import sys


def main(path, limit=None):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:limit + 1 if limit else None]:
        v = float(r[vi].replace(",", ""))
        v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(r[ui], v)
        name = r[ki].split("(")[0].replace("void ", "")
        name = name.split("rsvd::")[-1].replace("(anonymous namespace)::", "")[:58]
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':58s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:58s} {cnt[k]:8d} {v / 1e3:9.3f} {100 * v / s:5.1f}%")
    print(f"{'total':58s} {sum(cnt.values()):8d} {s / 1e3:9.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)

"""Top CUDA source lines by warp-stall samples from an ncu report (needs -lineinfo).

  python tools/ncu_source_hot.py gpurun_out/prof.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(path, n=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    res = []
    fname = None
    hdr = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Name":
            fname = r[1].split("/")[-1]
            hdr = None
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            try:
                v = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
            except (ValueError, IndexError):
                continue
            if v > 0:
                res.append((v, fname, r[0], r[1].strip()[:110]))
    tot = sum(x[0] for x in res) or 1.0
    res.sort(reverse=True)
    for v, f, ln, s in res[:n]:
        print(f"{100 * v / tot:5.1f}%  {f}:{ln}  {s}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)

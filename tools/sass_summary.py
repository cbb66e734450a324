"""Per-kernel SASS instruction counts of librsvd_b200.so (cuobjdump -sass):
the evidence that the GEMMs are TMA-fed (UTMALDG) and run on the FP64 tensor
pipe (DMMA) or, for the emulated-FP64 A-pass, on tcgen05 (UTCIMMA = tcgen05.mma
kind::i8, LDTM = tcgen05.ld), and which kernels use cp.async (LDGSTS), DSMEM / cluster
barriers, etc.  Usage: python tools/sass_summary.py [lib.so] > profiles/..."""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1710_01463_b200/librsvd_b200.so"
KEYS = ["DMMA", "UTCIMMA", "LDTM", "UTMALDG", "SYNCS", "LDGSTS", "DFMA", "MUFU", "BAR", "LDS", "LDG", "STG", "SHFL",
        "ATOM", "RED", "UCGABAR", "CCTL"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    cur, counts = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts.setdefault(cur, collections.Counter())
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
        if m:
            op = m.group(2)
            for k in KEYS:
                if op == k or op.startswith(k):
                    counts[cur][k] += 1
                    break
            counts[cur]["total"] += 1
    demangled = {}
    try:
        names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout
        demangled = dict(zip(counts, names.splitlines()))
    except OSError:
        pass
    print(f"# SASS summary of {LIB} (cuobjdump -sass; sm_100a)")
    print(f"{'kernel':70s} " + " ".join(f"{k:>7s}" for k in KEYS + ['total']))
    for fn, c in sorted(counts.items(), key=lambda kv: -kv[1]["DMMA"]):
        name = demangled.get(fn, fn)
        name = name.replace("(anonymous namespace)::", "").replace("void ", "")
        name = re.sub(r"\(.*", "", name).replace("rsvd::", "")[:70]
        print(f"{name:70s} " + " ".join(f"{c[k]:7d}" for k in KEYS + ['total']))


if __name__ == "__main__":
    main()

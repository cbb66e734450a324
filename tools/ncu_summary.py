"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

  python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/...txt
  python tools/ncu_summary.py report   gpurun_out/prof.ncu-rep  > profiles/...txt
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}


def launches(path, which="engine"):
    """which="engine": only the engine's kernels (rsvd:: namespace) -- the
    bench command also runs torch kernels that build the synthetic inputs."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        if which == "engine" and "rsvd::" not in r[ki] and "unnamed>::" not in r[ki]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.replace("rsvd::<unnamed>::", "")
        ms = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, "
          f"serialised): {sum(v[0] for v in agg.values())} launches, {tot:.2f} ms total")
    print(f"{'kernel':60s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {v[0]:8d} {v[1]:10.3f} {100 * v[1] / tot:6.1f}%")


METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        print(f"## {r[h.index('Kernel Name')][:110]}")
        for m in METRICS:
            if m in h:
                i = h.index(m)
                print(f"  {m:70s} {r[i]:>16s} {units[i]}")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](*sys.argv[2:])

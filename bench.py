#!/usr/bin/env python
"""FP64 RSVD truncations/sec on B200 (BASELINE.json metric).

Default workload: config C4 of BASELINE.json — a batch of 32 independent
4096 x 4096 FP64 bond matrices (chi=256, d=16), A = U diag(sigma) V^T with
Haar factors and sigma_i = exp(-0.02 i)(1 + 0.1 g_i), truncated to k=256 with
p=20 (l = 276) and q=2.  It is "4096^2, k=256", fits one GPU and shards by
item: at N GPUs the 32 matrices are split contiguously across the ranks (32/N
each, sharding.batch_partition), no collective on the data path -> scaling
"strong" (BASELINE: "batched across 8 GPUs"; `--weak` gives every rank its
own full batch instead).  `--gpus N` without torchrun re-launches itself
under torch.distributed.run with N ranks (127.0.0.1).

  value  : truncations/s over all ranks, inputs resident in HBM, device time
           (CUDA events on the launching stream, max over ranks).
  e2e    : same metric through the public API with pinned HOST buffers
           (H2D of A and D2H of U, S, Vt inside every timed step).
  roofline: the dominant kernel, the A-pass GEMM: on C4 / C5 the emulated-FP64
           INT8 tensor-core GEMM (ozaki.cu) against the measured tcgen05 kind::i8
           peak; on the smaller configs the DMMA GEMM against the measured FP64
           tensor peak.
  cpu_baseline: the reference's own rsvd (proj/src/factorize.cpp + lapack.cpp
           compiled unmodified into oracle/_ref/librlftn_ref.so, OpenBLAS
           LAPACK) on the host cores, rank 0 at N=1, on a bounded sample.

`--impl reference` times that same reference build on the same config with
all host threads.  Its process never touches CUDA or librsvd_b200.so: the
sample input is synthesised on the host (CounterRng Gaussians from the
reference's own generator, torch CPU QR), and the run checks its own
/proc/self/maps before printing.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

INT8_PEAK_TOPS = 8186 * 148 * 2 * 1.965e9 / 1e12  # tcgen05.mma kind::i8 rate, profiles/r02_umma_rate.txt
INT8_PEAK_SOURCE = ("measured tcgen05.mma.kind::i8 issue rate, 8186 MAC/clk/SM for N >= 128 "
                    "(profiles/r02_umma_rate.txt) x 148 SMs x 2 x the 1965 MHz max SM clock; "
                    "MEASURED_PEAKS.json has no INT8 figure")
def int8_vs_measured_bf16(achieved_tops):
    """Context for the INT8 roofline: MEASURED_PEAKS.json (driver-written) has the dense bf16
    cuBLAS throughput of this pool's B200s; INT8 tensor work runs at twice the bf16 rate, so
    2 x that figure is what a library GEMM would sustain under the same power limit."""
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        burst, sus = 2.0 * mp["bf16_tflops"], 2.0 * mp.get("bf16_tflops_sustained", mp["bf16_tflops"])
    except (OSError, ValueError, KeyError):
        return {}
    out = {"int8_tops_from_measured_bf16": {"burst": burst, "sustained": sus,
                                            "source": "2 x MEASURED_PEAKS.json bf16_tflops / bf16_tflops_sustained"}}
    if achieved_tops:
        out["frac_of_2x_measured_bf16_sustained"] = achieved_tops / sus
    return out


OZ_SLICE_PRODUCTS = 28  # 7 slices per operand, products p + q < 7 (ozaki.cu)
FP64_PEAK_TFLOPS = 37.1  # measured: mma.sync f64 probe, profiles/r01_fp64_peak.txt
FP64_PEAK_SOURCE = ("measured DMMA (mma.sync .f64) throughput on this pool's B200, "
                    "profiles/r01_fp64_peak.txt; MEASURED_PEAKS.json has no FP64 figure "
                    "(cuBLAS DGEMM 8192^3 measured 35.5)")


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def f_alg(m, n, k, ell, q):
    """LAPACK-nominal flops per truncation."""
    return (4 * (q + 1) * m * n * ell + 2 * m * ell * k
            + (q + 1) * (4 * m * ell ** 2 - 4 * ell ** 3 / 3)
            + q * (4 * n * ell ** 2 - 4 * ell ** 3 / 3) + 6 * n * ell ** 2 + 20 * ell ** 3)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        if os.environ.get("RSVD_BENCH_NO_CLOCKS"):  # diagnosis only
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None
        time.sleep(0.5)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        """Start of the timed region: only later samples are summarised.
        The sampler itself is started before the warm-up -- nvidia-smi's NVML
        initialisation stalled the first timed steps by up to 100 ms."""
        self.first = len(self.lines)

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        first = getattr(self, "first", 0)
        lines = self.lines[first:] if len(self.lines) > first else self.lines
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def make_inputs(cfg, items, first_item, device):
    from paper_1710_01463_b200 import synth

    return synth.make_batch(cfg, device=device, batch=items, first_item=first_item)


def cpu_checker():
    """The reference build (oracle/_ref/librlftn_ref.so) when present -- kind
    "reference" -- else the restatement port (bitwise equal to it,
    tests/test_ref_pin_cpu.py) -- kind "port"."""
    from oracle import oracle, ref

    if ref.available():
        return ref, "reference", ("reference rsvd: proj/src/factorize.cpp + lapack.cpp compiled "
                                  "unmodified (oracle/_ref), OpenBLAS 0.3.31 LAPACK")
    return oracle, "port", "oracle rsvd (restated reference, OpenBLAS 0.3.31 LAPACK)"


def cpu_ref_rsvd(A_items, cfg, seeds, threads):
    """Time the reference rsvd on host copies of the given items; returns
    (seconds per truncation list)."""
    mod, _, _ = cpu_checker()
    mod.set_threads(threads)
    times = []
    for a, s in zip(A_items, seeds):
        t0 = time.perf_counter()
        mod.rsvd(a, cfg.rank, cfg.ell, cfg.power, s)
        times.append(time.perf_counter() - t0)
    return times


L2_BYTES = 126 * 1024 * 1024  # B200 L2


def l2_flush_buffer(input_bytes, dev):
    """A 256 MB device buffer to overwrite before every timed step when the
    per-rank inputs are under twice the L2 (C1 8 MB, C2/C3 134 MB), else None
    (C4 4.3 GB, C5 537 MB: the inputs themselves stream through L2)."""
    import torch

    if input_bytes >= 2 * L2_BYTES:
        return None
    return torch.empty(2 * L2_BYTES // 8, dtype=torch.float64, device=dev)


def l2_note(input_bytes):
    if input_bytes >= 2 * L2_BYTES:
        return "inputs larger than L2 (%.2f GB per rank, > 2 x 126 MB)" % (input_bytes / 1e9)
    return ("L2 flushed before every timed step (252 MB write outside the timed span; "
            "inputs %.1f MB per rank)" % (input_bytes / 1e6))


def cpu_modes(A_items, cfg, seeds, threads, budget_s):
    """the reference protocol (1 BLAS thread) and all host cores,
    for both methods -- rsvd and full-SVD truncation (tsvd = dgesdd +
    truncate) -- on the first matrix of the sample; each mode is skipped once
    the accumulated CPU time passes `budget_s`."""
    mod, _, _ = cpu_checker()
    a, s = A_items[0], seeds[0]
    out, spent = {}, 0.0
    for name, fn, th in (("rsvd_1thread", lambda: mod.rsvd(a, cfg.rank, cfg.ell, cfg.power, s), 1),
                         ("rsvd_all_cores", lambda: mod.rsvd(a, cfg.rank, cfg.ell, cfg.power, s), threads),
                         ("tsvd_all_cores", lambda: mod.tsvd(a, cfg.rank), threads),
                         ("tsvd_1thread", lambda: mod.tsvd(a, cfg.rank), 1)):
        if spent > budget_s:
            out[name] = None
            continue
        mod.set_threads(th)
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        spent += dt
        out[name] = {"value": 1.0 / dt, "unit": "truncations/s", "cores": th}
    mod.set_threads(threads)
    return out


METRIC = "FP64 RSVD truncations/sec (4096^2, k=256)"
DATA = "synthetic (BASELINE.json config recipe, seeded CounterRng, Haar factors)"


def batch_config(cfg, world, count_per_rank, global_batch, weak):
    """The `config` object of a batch-split line -- shared verbatim by the GPU
    arm and the reference arm (same workload, same N)."""
    return {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "batch_per_rank": count_per_rank,
            "global_batch": global_batch, "rank_k": cfg.rank, "ell": cfg.ell,
            "power_q": cfg.power,
            "parallelism": (f"batch replicated dp{world} (weak)" if weak
                            else f"batch split dp{world}"),
            "l2": l2_note(count_per_rank * cfg.m * cfg.n * 8)}


def rowshard_config(cfg, world, rows_per_rank):
    return {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "rank_k": cfg.rank,
            "ell": cfg.ell, "power_q": cfg.power,
            "parallelism": f"row shard x{world} (NCCL all-reduce of Grams / A^T Q panels)",
            "rows_per_rank": rows_per_rank, "l2": l2_note(rows_per_rank * cfg.n * 8)}


def rowsharded(args, world, cfg):
    return args.rowshard or (world > 1 and cfg.batch == 1)


def loaded_shared_objects():
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")
                           or ".so." in ln})
    except OSError:
        return []


def run_reference(args, rank, world):
    """The reference's own rsvd (oracle/_ref: proj/src/factorize.cpp + lapack.cpp
    compiled unmodified) on the host cores, on the GPU arm's config.  Rank 0
    alone runs under torchrun; CUDA and librsvd_b200.so are never touched."""
    if rank != 0:
        return 0
    import numpy as np
    import torch

    from paper_1710_01463_b200 import sharding, synth

    mod, kind, what = cpu_checker()
    cfg = synth.CONFIGS[args.config]
    threads = host_threads()
    sample = max(1, args.ref_sample)
    # the GPU arm's workload description at this N (verbatim)
    if rowsharded(args, world, cfg):
        config = rowshard_config(cfg, world, sharding.row_partition(cfg.m, world, 0)[1])
        units = 1
    else:
        glob = cfg.batch if args.batch is None else args.batch
        per = glob if args.weak else sharding.batch_partition(glob, world, 0)[1]
        config = batch_config(cfg, world, per, glob * world if args.weak else glob, args.weak)
        units = config["global_batch"]
    # host-side synthesis of the sample: the reference's own CounterRng
    # Gaussians (the same streams the GPU arm draws on the device) + torch CPU QR
    gauss = lambda seed, count: torch.from_numpy(mod.fill_gaussian(seed, count))  # noqa: E731
    mats = [np.asfortranarray(synth.make_matrix(cfg, i, "cpu", gauss).numpy())
            for i in range(min(sample, cfg.batch))]
    seeds = synth.omega_seeds(cfg, batch=len(mats))
    for _ in range(args.warmup):
        cpu_ref_rsvd(mats[:1], cfg, seeds[:1], threads)
    t = 0.0
    for _ in range(args.steps):
        t += sum(cpu_ref_rsvd(mats, cfg, seeds, threads))
    value = args.steps * len(mats) / t
    one = None
    if args.ref_one_thread:
        one = 1.0 / sum(cpu_ref_rsvd(mats[:1], cfg, seeds[:1], 1))
        mod.set_threads(threads)
    sos = loaded_shared_objects()
    bad = [p for p in sos if "librsvd_b200" in p]
    if bad or torch.cuda.is_initialized():
        raise SystemExit(f"reference arm touched the GPU path: {bad}")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value, "unit": "truncations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * t / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": config,
        "reference_sample": {
            "step": f"{len(mats)} of the {units} truncation(s) of the workload per step "
                    "(bounded CPU sample; value = truncations per second of CPU time)",
            "input": "host-synthesised (reference CounterRng Gaussians, torch CPU QR)"},
        "cpu_baseline": {"value": value, "unit": "truncations/s", "cores": threads,
                         "kind": kind, "sample": f"{len(mats)} {cfg.m}x{cfg.n} matrix per step, "
                                                 + what + ", all host threads",
                         "rsvd_1thread": (None if one is None else
                                          {"value": one, "unit": "truncations/s", "cores": 1,
                                           "note": "reference protocol: BLAS pinned to one "
                                                   "thread (lapack.cpp:225, main.cpp:7)"})},
        "e2e": {"value": value, "unit": "truncations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "loaded_native": [p for p in sos if "/oracle/" in p],
    }
    print(json.dumps(line))
    return 0


def run_rowsharded(args, rank, world, local_rank):
    """One large matrix (C3 / C5) row-sharded over `world` GPUs: NCCL all-reduce
    of the l x l Grams and n x l panels only; strong scaling (fixed problem)."""
    import torch
    import torch.distributed as dist

    from paper_1710_01463_b200 import Handle, RsvdParams, _lib, sharding, synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS[args.config]
    A = synth.make_matrix(cfg, 0, dev)  # identical on every rank (same seeds)
    first, count = sharding.row_partition(cfg.m, world, rank)
    a_loc = A[first:first + count].t().contiguous().t()
    del A
    torch.cuda.empty_cache()
    seed = synth.omega_seed(cfg, 0)
    params = RsvdParams(cfg.rank, cfg.ell, cfg.power, seed)
    h = Handle(local_rank)
    sharding.attach_nccl(h, world, rank)
    clocks = ClockSampler(local_rank)
    clocks.start()
    for _ in range(args.warmup):
        sharding.rsvd_rowsharded(a_loc, cfg.m, first, params, h)
    torch.cuda.synchronize()
    clocks.mark()
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    flush = l2_flush_buffer(count * cfg.n * 8, dev)
    pairs = []
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es.record()
        f = sharding.rsvd_rowsharded(a_loc, cfg.m, first, params, h)
        ee.record()
        pairs.append((es, ee))
    torch.cuda.synchronize()
    step_ms = sum(a.elapsed_time(b) for a, b in pairs)
    dist.barrier()
    launches = _lib.kernel_launches() - launches0
    clk = clocks.stop()
    t = torch.tensor([step_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = args.steps / (ms / 1000.0)
    # e2e: this rank's row block from pinned host memory, factors back to the host
    a_host = torch.empty_strided(a_loc.shape, a_loc.stride(), dtype=a_loc.dtype, pin_memory=True)
    a_host.copy_(a_loc)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        a_dev = a_host.to(dev, non_blocking=True)
        fe = sharding.rsvd_rowsharded(a_dev, cfg.m, first, params, h)
        _ = (fe.left.cpu(), fe.sigma.cpu(), fe.right_adj.cpu())
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = args.steps / float(te.item())
    if rank == 0:
        falg = f_alg(cfg.m, cfg.n, cfg.rank, cfg.ell, cfg.power)
        k = cfg.rank
        print(json.dumps({
            "metric": METRIC,
            "value": value, "unit": "truncations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": rowshard_config(cfg, world, sharding.row_partition(cfg.m, world, 0)[1]),
            "e2e": {"value": e2e_value, "unit": "truncations/s",
                    "h2d_bytes_per_step": count * cfg.n * 8,
                    "d2h_bytes_per_step": (count * k + k + k * cfg.n) * 8},
            "gpu_launches": launches,
            "pipeline": {"tflops_alg": falg * value / 1e12, "rank_out": f.rank()},
            "clocks": clk,
        }))
    dist.destroy_process_group()
    return 0


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1710_01463_b200 import Handle, RsvdParams, _lib, rsvd_batched, sharding, synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = synth.CONFIGS[args.config]
    glob = cfg.batch if args.batch is None else args.batch
    if args.weak:  # every rank its own full batch (opt-in)
        B, first, total = glob, rank * glob, glob * world
    else:          # BASELINE: the batch is split across the GPUs (strong)
        first, B = sharding.batch_partition(glob, world, rank)
        total = glob
    if B < 1:
        raise SystemExit(f"rank {rank}: no items ({glob} over {world} ranks)")
    A = make_inputs(cfg, B, first, dev)
    seeds = synth.omega_seeds(cfg, batch=B, first_item=first)
    params = RsvdParams(cfg.rank, cfg.ell, cfg.power, 0)
    h = Handle(local_rank)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local_rank)
    clocks.start()
    # Factors are written into the same device buffers every step (out=): a
    # fresh 0.5 GB allocation per step made the second timed step re-allocate
    # and re-capture its CUDA graph (+3 .. +100 ms).
    f = None
    for _ in range(args.warmup):
        f = rsvd_batched(A, params, seeds, handle=h, out=f)
    torch.cuda.synchronize()

    # ---- device-resident timed region --------------------------------
    clocks.mark()
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.kernel_launches()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    verbose = bool(os.environ.get("RSVD_BENCH_VERBOSE"))
    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] if verbose else []
    host_t = []
    flush = l2_flush_buffer(B * cfg.m * cfg.n * 8, dev)
    if flush is None:
        e0.record(stream)
        for i in range(args.steps):
            th = time.perf_counter()
            f = rsvd_batched(A, params, seeds, handle=h, out=f)
            if verbose:
                step_ev[i].record(stream)
                host_t.append(round((time.perf_counter() - th) * 1e3, 2))
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms = e0.elapsed_time(e1)
    else:
        # Inputs fit the 126 MB L2: flush it before every step, time the steps only.
        pairs = []
        for i in range(args.steps):
            flush.zero_()
            es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            es.record(stream)
            f = rsvd_batched(A, params, seeds, handle=h, out=f)
            ee.record(stream)
            pairs.append((es, ee))
        torch.cuda.synchronize()
        step_ms = sum(a.elapsed_time(b) for a, b in pairs)
    if verbose:
        prev, dev_t = e0, []
        for ev in step_ev:
            dev_t.append(round(prev.elapsed_time(ev), 2))
            prev = ev
        print("step device ms:", dev_t, "host ms:", host_t, file=sys.stderr)
    barrier()
    launches = _lib.kernel_launches() - launches0
    clk = clocks.stop()
    ms = max_over_ranks(step_ms)
    value = total * args.steps / (ms / 1000.0)
    ranks_ok = all(r == cfg.rank for r in f.ranks)

    # ---- per-stage profile pass (events around each stage) ------------
    _lib.profile_enable(h, True)
    prof_steps = max(1, min(2, args.steps))
    for _ in range(prof_steps):
        rsvd_batched(A, params, seeds, handle=h)
    torch.cuda.synchronize()
    prof = _lib.profile_read(h)
    _lib.profile_enable(h, False)
    sweeps = _lib.last_jacobi_sweeps(h)
    # GPU full-SVD truncation (tsvd, factorize.cpp:42-50), the comparator the
    # BASELINE configs name: the whole rank's batch when min(m, n) <= 1600,
    # otherwise one item of it (a full SVD of 4096^2 / 32768 x 2048 per call).
    gpu_tsvd = None
    if not args.no_gpu_tsvd:
        from paper_1710_01463_b200 import tsvd_batched

        nt = B if min(cfg.m, cfg.n) <= 1600 else 1
        At = A[:nt]
        ft = tsvd_batched(At, cfg.rank, handle=h)
        torch.cuda.synchronize()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0e.record(stream)
        ft = tsvd_batched(At, cfg.rank, handle=h)
        t1e.record(stream)
        torch.cuda.synchronize()
        tms = max_over_ranks(t0e.elapsed_time(t1e))
        gpu_tsvd = {"value": nt * world / (tms / 1000.0), "unit": "truncations/s", "ms_per_call": tms,
                    "items_per_call": nt,
                    "note": "tsvd_batched: CholeskyQR3 of A^T + one-sided Jacobi on the full "
                            "min(m, n) factor (row-streamed dataflow / cluster kernels), 1 call"}
        del ft, At
    gemm_path = _lib.last_gemm_path(h)
    slice_ms = prof.get("apass_slice", (0.0, 0))[0]  # nested inside the A-pass stages
    ap_ms = prof["apass_nn"][0] + prof["apass_tn"][0]
    ap_calls = prof["apass_nn"][1] + prof["apass_tn"][1]
    gemm_ms = ap_ms - slice_ms
    ap_flops_per_launch = 2.0 * cfg.m * cfg.n * cfg.ell * B  # algorithmic: one pass over A per item
    fp64_equiv = ap_flops_per_launch / (gemm_ms / ap_calls / 1000.0) / 1e12 if ap_calls else None
    step_ms_prof = (sum(v[0] for v in prof.values()) - slice_ms) / prof_steps
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(tpath):
        try:
            key = "oz_gemm_dram_bytes_per_launch" if gemm_path == "ozaki" else "apass_dram_bytes_per_launch"
            traffic = json.load(open(tpath)).get(key)
        except (OSError, ValueError):
            traffic = None
    if gemm_path == "ozaki":
        ops_per_launch = OZ_SLICE_PRODUCTS * ap_flops_per_launch  # INT8 ops of the slice products
        achieved = ops_per_launch / (gemm_ms / ap_calls / 1000.0) / 1e12 if ap_calls else None
        roof = {"bound": "tensor", "achieved": achieved, "peak": INT8_PEAK_TOPS, "unit": "TOP/s",
                "frac": (achieved / INT8_PEAK_TOPS) if achieved else None, "traffic": traffic,
                "kernel": "oz_gemm_kernel A-pass (Y=A X / Z=A^T Y): FP64 emulated from 7 x 7 "
                          "signed 8-bit slices on tcgen05.mma.kind::i8, TMA-fed, TMEM accumulators",
                "algorithmic_ops_per_launch": ops_per_launch,
                "algorithmic_fp64_flops_per_launch": ap_flops_per_launch,
                "fp64_equivalent_tflops": fp64_equiv,
                "fp64_equivalent_vs_dmma_peak": (fp64_equiv / FP64_PEAK_TFLOPS) if fp64_equiv else None,
                "peak_source": INT8_PEAK_SOURCE,
                "slice_ms_per_step": slice_ms / prof_steps,
                **int8_vs_measured_bf16(achieved),
                "apass_share_of_step": gemm_ms / prof_steps / step_ms_prof}
    else:
        roof = {"bound": "tensor", "achieved": fp64_equiv, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s",
                "frac": (fp64_equiv / FP64_PEAK_TFLOPS) if fp64_equiv else None,
                "traffic": traffic,
                "kernel": "dgemm_tma_kernel A-pass (Y=A X / Z=A^T Y; TMA-fed DMMA), batched over the step",
                "algorithmic_flops_per_launch": ap_flops_per_launch,
                "peak_source": FP64_PEAK_SOURCE,
                "apass_share_of_step": gemm_ms / prof_steps / step_ms_prof}

    # ---- end-to-end through the public API with pinned host buffers ---
    try:
        A_host = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype, pin_memory=True)
        e2e_pinned = True
    except RuntimeError:  # host out of page-locked memory (N ranks x 4.3 GB): pageable fallback
        A_host = torch.empty_strided(A.shape, A.stride(), dtype=A.dtype)
        e2e_pinned = False
    A_host.copy_(A)
    del A
    torch.cuda.empty_cache()
    # warm the host-path workspace; its pinned factors are reused via out=
    fe = rsvd_batched(A_host, params, seeds, handle=h)
    barrier()
    t0 = time.perf_counter()
    per_call = []
    for _ in range(args.steps):
        tc = time.perf_counter()
        fe = rsvd_batched(A_host, params, seeds, handle=h, out=fe)
        _ = fe.sigma[0, 0].item()  # result read on the host
        per_call.append(round((time.perf_counter() - tc) * 1e3, 1))
    t_e2e = max_over_ranks(time.perf_counter() - t0)
    if os.environ.get("RSVD_BENCH_VERBOSE"):
        print("e2e per call ms:", per_call, file=sys.stderr)
    e2e_value = total * args.steps / t_e2e
    k = max(cfg.rank, 1)
    h2d = B * cfg.m * cfg.n * 8 + B * 8
    d2h = B * (cfg.m * k + k + k * cfg.n) * 8 + B * 16

    # ---- CPU baseline (rank 0, N=1) -----------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_threads()
        n_cpu = max(1, args.cpu_sample)
        mats = [np.asfortranarray(A_host[i].numpy()) for i in range(min(n_cpu, B))]
        times = cpu_ref_rsvd(mats, cfg, seeds[:len(mats)], threads)
        _, kind, what = cpu_checker()
        cpu = {"value": len(times) / sum(times), "unit": "truncations/s", "cores": threads,
               "kind": kind,
               "sample": f"{len(times)} of the {B} {cfg.m}x{cfg.n} matrices, {what}, "
                         "all host threads"}
        cpu["modes"] = cpu_modes(mats, cfg, seeds, threads, args.cpu_modes_budget)
        cpu["modes"]["sample"] = (f"item 0 ({cfg.m}x{cfg.n}); a mode is skipped (null) once "
                                  f"{args.cpu_modes_budget:.0f} s of CPU time were spent")

    if rank == 0:
        falg = f_alg(cfg.m, cfg.n, cfg.rank, cfg.ell, cfg.power)
        line = {
            "metric": METRIC,
            "value": value, "unit": "truncations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": batch_config(cfg, world, B, total, args.weak),
            "e2e": {"value": e2e_value, "unit": "truncations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "host_memory": "pinned" if e2e_pinned else "pageable"},
            "gpu_launches": launches,
            "roofline": roof,
            "gemm_path": gemm_path,
            "precision": ("f64 in and out; A-pass products rebuilt exactly from 7 x 7 signed 8-bit "
                          "slice products (54-bit operands, INT32 / FP64 accumulation): elementwise "
                          "within 8e-15 |A||B| of torch f64 (tests/test_gpu_kernels.py), parity with "
                          "the reference build at this size in tests/test_gpu_configs.py"
                          if gemm_path == "ozaki" else "f64 (DMMA) throughout"),
            "pipeline": {"tflops_alg": falg * total * args.steps / (ms / 1000) / 1e12 / world,
                         "frac_fp64_peak": falg * B * args.steps / (ms / 1000) / 1e12 / FP64_PEAK_TFLOPS,
                         "stage_ms_per_step": {k2: v[0] / prof_steps for k2, v in prof.items()},
                         "jacobi_sweeps": sweeps, "ranks_ok": ranks_ok},
            "clocks": clk,
        }
        if gpu_tsvd is not None:
            line["gpu_tsvd"] = gpu_tsvd
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn(args) -> int:
    """`--gpus N` outside torchrun: re-launch this script as N ranks (one per
    GPU) under torch.distributed.run on 127.0.0.1, as the driver does."""
    import socket

    if args.impl != "reference":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} GPU(s) visible", file=sys.stderr)
            return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--batch", type=int, default=None, help="override the global batch")
    ap.add_argument("--weak", action="store_true",
                    help="every rank factorizes its own full batch (weak scaling)")
    ap.add_argument("--cpu-sample", type=int, default=2)
    ap.add_argument("--ref-sample", type=int, default=1)
    ap.add_argument("--ref-one-thread", action=argparse.BooleanOptionalAction, default=True,
                    help="reference arm: also time one truncation with 1 BLAS thread")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gpu-tsvd", action="store_true", help="skip the GPU full-SVD comparator")
    ap.add_argument("--cpu-modes-budget", type=float, default=45.0,
                    help="seconds of CPU time for the 1-thread / tsvd baseline modes")
    ap.add_argument("--rowshard", action="store_true",
                    help="row-sharded single-matrix path (default for C3/C5 when N > 1)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":
            return run_reference(args, 0, args.gpus)
        return spawn(args)
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    from paper_1710_01463_b200 import synth

    if rowsharded(args, world, synth.CONFIGS[args.config]):
        return run_rowsharded(args, rank, world, local_rank)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())

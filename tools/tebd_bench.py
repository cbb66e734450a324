"""TEBD layer throughput: one imaginary-time layer of two-site gates on a
spin chain at bond dimension chi, GPU (apply_gate_layer: one batched
factorization for all bonds of the layer, and gate-by-gate apply_gate) against
the CPU oracle (oracle/tebd_oracle.py over the restated LAPACK path, all host
cores).  Prints one JSON line.

    python tools/tebd_bench.py [--length 64] [--chi 256] [--method rsvd|tsvd]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1710_01463_b200 import BlockMethod, RankPolicy, SectorRankRequest  # noqa: E402
from tests import tebd_helpers as TH
from tests import tebd_models as M  # noqa: E402
from paper_1710_01463_b200 import tebd  # noqa: E402


def random_mps(site, length, chi, dev):
    """A synthetic Gamma/lambda state at full bond dimension: sector sizes
    min(chi / 2, d^j / 2, d^(L-j) / 2), Gaussian Gamma blocks, decaying
    normalised lambdas (the load of a saturated TEBD run; not a physical
    state)."""
    g = torch.Generator().manual_seed(5)
    d = site.dim
    half = []
    for b in range(length + 1):
        cap = min(chi // 2, (d ** min(b, length - b)) // 2 if min(b, length - b) < 20 else chi)
        half.append(max(cap, 0))
    lambdas = []
    for b in range(length + 1):
        if b in (0, length):
            lambdas.append([torch.ones(1, dtype=torch.float64, device=dev),
                            torch.zeros(0, dtype=torch.float64, device=dev)])
            continue
        n = half[b]
        v = torch.exp(-0.05 * torch.arange(2 * n, dtype=torch.float64))
        v = v / torch.linalg.norm(v)
        lambdas.append([v[0::2].to(dev), v[1::2].to(dev)])
    gammas = []
    for j in range(length):
        st = []
        for m in range(d):
            pair = []
            for a in (0, 1):
                r = lambdas[j][a].numel()
                c = lambdas[j + 1][a ^ site.charges[m]].numel()
                pair.append(torch.randn(r, c, generator=g, dtype=torch.float64).to(dev))
            st.append(pair)
        gammas.append(st)
    return tebd.SymmetricMPS(site, gammas, lambdas)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--length", type=int, default=64)
    ap.add_argument("--chi", type=int, default=256)
    ap.add_argument("--method", default="rsvd")
    ap.add_argument("--dt", type=float, default=0.1)
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--cpu-bonds", type=int, default=4)
    ap.add_argument("--random-state", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    model = M.ChainModel(args.length, 0.5, 1.0)
    site = M.parity_structure(model)
    hs = M.bond_hamiltonians(model)
    gates = [M.build_gate(h, site.charges, args.dt) for h in hs]
    meth = BlockMethod.randomized(4, 7) if args.method == "rsvd" else BlockMethod.deterministic()
    req = SectorRankRequest(RankPolicy.per_sector_estimate, 0)
    layers = [list(range(0, args.length - 1, 2)), list(range(1, args.length - 1, 2))]
    if args.random_state:
        psi = random_mps(site, args.length, args.chi, dev)
    else:
        psi = TH.random_product_state(site, args.length, 1, device=dev)
        # grow the entanglement (imaginary time saturates well below chi on
        # the critical chain; --random-state loads the full chi instead)
        for i in range(64):
            lay = layers[i % 2]
            tebd.apply_gate_layer(psi, lay, [gates[b] for b in lay], args.chi, meth, req)
            if psi.max_bond_dimension() >= args.chi and i >= 16:
                break
    torch.cuda.synchronize()

    def run_layers(batched):
        t0 = time.perf_counter()
        for i in range(args.layers):
            lay = layers[i % 2]
            if batched:
                tebd.apply_gate_layer(psi, lay, [gates[b] for b in lay], args.chi, meth, req)
            else:
                for b in lay:
                    tebd.apply_gate(psi, b, gates[b], args.chi, meth, req)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / args.layers

    run_layers(True)
    t_batched = run_layers(True)
    t_seq = run_layers(False)
    bonds_per_layer = sum(len(layers[i % 2]) for i in range(args.layers)) / args.layers

    # CPU oracle on a bounded number of bonds of one layer (same state)
    from oracle import oracle as O
    from oracle import tebd_oracle

    O.set_threads(os.cpu_count() or 1)
    g, lam = psi.to_numpy()
    mid = len(layers[0]) // 2  # middle bonds (full chi), not the thin chain ends
    lay = layers[0][max(0, mid - args.cpu_bonds // 2):][:args.cpu_bonds]
    t0 = time.perf_counter()
    for b in lay:
        tebd_oracle.apply_gate(g, lam, site.charges, b, gates[b].block, None, "block", args.chi,
                               kind=args.method, power=4, seed=7)
    t_cpu_bond = (time.perf_counter() - t0) / len(lay)
    line = {
        "metric": "TEBD two-site gates/s (imaginary-time layer, Z2 spin-1/2 chain)",
        "config": {"length": args.length, "chi": args.chi, "method": args.method,
                   "max_bond": psi.max_bond_dimension(), "bonds_per_layer": bonds_per_layer,
                   "mean_bond": float(np.mean([psi.bond_dimension(b) for b in range(args.length + 1)])),
                   "state": "random saturated Gamma/lambda" if args.random_state else "imaginary-time evolved"},
        "gpu_layer_batched": {"value": bonds_per_layer / t_batched, "unit": "gates/s",
                              "ms_per_layer": t_batched * 1e3},
        "gpu_gate_by_gate": {"value": bonds_per_layer / t_seq, "unit": "gates/s",
                             "ms_per_layer": t_seq * 1e3},
        "cpu_oracle": {"value": 1.0 / t_cpu_bond, "unit": "gates/s", "cores": os.cpu_count(),
                       "sample": f"{len(lay)} middle bonds (dims {[psi.bond_dimension(b + 1) for b in lay]}) of one layer, gate by gate"},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()

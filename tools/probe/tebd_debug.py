"""Reproduce test_apply_gate_vs_oracle[tsvd-block] and inspect the failing bond."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1710_01463_b200 import models as M, tebd, BlockMethod, RankPolicy, SectorRankRequest, tsvd
from tests.test_gpu_tebd import _entangled

cuda = torch.device("cuda:0")
m = M.ChainModel(8, 1.0, 1.2)
st, g, lam, psi = _entangled(m, 40, 0.3, 4, 41, cuda)
bonds = M.bond_hamiltonians(m)
meth = BlockMethod.deterministic()
meth.rsvd_min_dim = 8
req = SectorRankRequest(RankPolicy.per_sector_estimate, 24)
for ps in range(2):
    for b in range(ps % 2, m.length - 1, 2):
        gate = M.build_gate(bonds[b], st.charges, 0.2)
        plan = tebd._assemble(psi, b, gate)
        for s, A in enumerate(plan.thetap):
            if A.numel() == 0:
                continue
            a = A.cpu().numpy()
            sv = np.linalg.svd(a, compute_uv=False)
            f = tsvd(A, 200)
            sg = f.sigma.cpu().numpy()
            tot = float(np.sum(a * a))
            print(f"bond {b} sector {s} shape {a.shape} rank_np {np.sum(sv > sv[0]*1e-14)} rank_gpu {len(sg)} "
                  f"1-sum/tot gpu {1 - np.sum(sg**2)/tot:.3e} np {1 - np.sum(sv**2)/tot:.3e} "
                  f"maxrel(top) {np.max(np.abs(sg[:10]-sv[:10])/sv[:10]):.2e} dw {f.discarded_weight:.3e}")
        tebd.apply_gate(psi, b, gate, 24, meth, req)

# detail of a bond-3 style block: rebuild the state and print spectra
st, g, lam, psi = _entangled(m, 40, 0.3, 4, 41, cuda)
for ps in range(2):
    for b in range(ps % 2, m.length - 1, 2):
        gate = M.build_gate(bonds[b], st.charges, 0.2)
        if b == 3:
            plan = tebd._assemble(psi, b, gate)
            A = plan.thetap[0]
            a = A.cpu().numpy()
            sv = np.linalg.svd(a, compute_uv=False)
            f = tsvd(A, 200)
            sg = f.sigma.cpu().numpy()
            np.set_printoptions(precision=6, linewidth=200)
            print("numpy:", sv[:16])
            print("gpu  :", sg[:16])
            fT = tsvd(A.t().contiguous(), 200)
            print("gpuT :", fT.sigma.cpu().numpy()[:16])
            np.save("gpurun_out/theta_b3.npy", a)
            raise SystemExit
        tebd.apply_gate(psi, b, gate, 24, meth, req)

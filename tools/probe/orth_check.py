"""Orthogonality / residual of the final factors on the bench configs:
max |U^T U - I|, max |V^T V - I| and ||A - U S V^T||_F / ||A||_F per item, for
the package found first on sys.path (PYTHONPATH selects a build to compare).
    python tools/probe/orth_check.py [C1 C2 ...]"""
import os
import sys

sys.path.append(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1710_01463_b200 import RsvdParams, rsvd_batched, synth  # noqa: E402
import paper_1710_01463_b200 as pkg  # noqa: E402

print("package:", os.path.dirname(pkg.__file__))
for c in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    cfg = synth.CONFIGS[c]
    A = synth.make_batch(cfg, device="cuda:0")
    f = rsvd_batched(A, RsvdParams(cfg.rank, cfg.ell, cfg.power, 0), synth.omega_seeds(cfg))
    ou = ov = res = 0.0
    for b in range(A.shape[0]):
        r = int(f.ranks[b])
        U, S, Vh = f.left[b][:, :r], f.sigma[b][:r], f.right_adj[b][:r, :]
        I = torch.eye(r, dtype=U.dtype, device=U.device)
        ou = max(ou, (U.T @ U - I).abs().max().item())
        ov = max(ov, (Vh @ Vh.T - I).abs().max().item())
        res = max(res, (torch.linalg.norm(A[b] - (U * S) @ Vh) / torch.linalg.norm(A[b])).item())
    print(f"{c}: max|UtU-I| {ou:.2e}  max|VVt-I| {ov:.2e}  max rel residual {res:.6e}")
    del A, f
    torch.cuda.empty_cache()

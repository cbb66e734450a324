import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1710_01463_b200 import _lib as L, tsvd
h = L.default_handle()
for (m, n) in [(300, 96), (300, 90), (256, 50), (600, 96), (1024, 74), (1024, 96), (301, 40), (5000, 160), (3, 3), (17, 3)]:
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    X = torch.from_numpy(a.T.copy()).cuda().t()
    Q = torch.empty((n, m), dtype=torch.float64, device="cuda").t()
    R = torch.empty((n, n), dtype=torch.float64, device="cuda").t()
    L.raise_for(L.load().rsvd_qr_f64(h.raw, 1, X.data_ptr(), m, n, m, m * n, Q.data_ptr(), m, m * n,
                                     R.data_ptr(), n, n * n, L.PTR_DEVICE), h.raw)
    torch.cuda.synchronize()
    q, r = Q.cpu().numpy(), R.cpu().numpy()
    print((m, n), "orth %.2e" % np.abs(q.T @ q - np.eye(n)).max(), "RtR-G %.2e" % np.abs(r.T @ r - a.T @ a).max())

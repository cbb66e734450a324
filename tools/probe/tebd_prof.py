"""cProfile of apply_gate_layer at small chi (where host overhead dominates)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

sys.argv = [sys.argv[0], "--chi", "32", "--random-state"]
import tools.tebd_bench as tb  # noqa: E402
from paper_1710_01463_b200 import BlockMethod, RankPolicy, SectorRankRequest, tebd  # noqa: E402
from paper_1710_01463_b200 import models as M  # noqa: E402

dev = torch.device("cuda:0")
model = M.ChainModel(64, 0.5, 1.0)
site = M.parity_structure(model)
gates = [M.build_gate(h, site.charges, 0.1) for h in M.bond_hamiltonians(model)]
psi = tb.random_mps(site, 64, 32, dev)
meth = BlockMethod.randomized(4, 7)
req = SectorRankRequest(RankPolicy.per_sector_estimate, 0)
lay = list(range(0, 63, 2))
tebd.apply_gate_layer(psi, lay, [gates[b] for b in lay], 32, meth, req)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(4):
    lay = list(range(i % 2, 63, 2))
    tebd.apply_gate_layer(psi, lay, [gates[b] for b in lay], 32, meth, req)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

"""cProfile of one TEBD layer (host orchestration breakdown)."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.argv = [sys.argv[0]] + sys.argv[1:]
import torch
from tools import tebd_bench as TB
from paper_1710_01463_b200 import BlockMethod, RankPolicy, SectorRankRequest, tebd
from tests import tebd_models as M
chi = int(os.environ.get("CHI", "32"))
dev = torch.device("cuda:0")
model = M.ChainModel(64, 0.5, 1.0)
site = M.parity_structure(model)
gates = [M.build_gate(h, site.charges, 0.1) for h in M.bond_hamiltonians(model)]
meth = BlockMethod.randomized(4, 7)
req = SectorRankRequest(RankPolicy.per_sector_estimate, 0)
psi = TB.random_mps(site, 64, chi, dev)
lay = list(range(0, 63, 2))
for _ in range(3):
    tebd.apply_gate_layer(psi, lay, [gates[b] for b in lay], chi, meth, req)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(5):
    tebd.apply_gate_layer(psi, lay, [gates[b] for b in lay], chi, meth, req)
torch.cuda.synchronize()
pr.disable()
print("ms per layer", (time.perf_counter() - t0) / 5 * 1e3)
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)

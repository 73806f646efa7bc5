"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck): heavy and light roots,
k = 3 and 4, directed and undirected, forced paths, slices, edge counts, NCCL-free.
python tools/sanitize_case.py [quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
g = G.make_config("cfg3", scale=0.0025 if quick else 0.008)   # hubs of G_U degree > 128 + light roots
n, s, d = g
deg = np.bincount(np.concatenate([s, d]), minlength=n)
print(f"n={n} arcs={s.size} max degree {deg.max()} heavy roots {(deg > 128).sum()}", flush=True)
gr = vdmc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
tot = {}
for k in (3, 4):
    for kind in ("directed", "undirected"):
        out = gr.count(k, kind=kind)
        tot[(k, kind)] = int(out.sum().item())
opts = [{"heavy_global": 1}, {"heavy_global": 1, "force_big": 1}, {"star_block": 1023},
        {"ca_capacity": 3, "star_block": 7, "cross_block": 32, "force_big": 1}]   # closed forms + enumerated path
for o in opts:
    assert int(gr.count(4, options=o).sum().item()) == tot[(4, "directed")], o
acc = None
for sl in gr.plan(4, 3):
    x = gr.count(4, work=sl)
    acc = x if acc is None else acc + x
assert int(acc.sum().item()) == tot[(4, "directed")]
e = gr.count_edges(4)
print("edges", e.shape, int(e.sum().item()), flush=True)
rk = np.random.default_rng(1).permutation(n)
g2 = vdmc.Graph(n, s, d, rank=rk)
assert int(g2.count(4).sum().item()) == tot[(4, "directed")]
torch.cuda.synchronize()
print("sanitize case ok", tot, flush=True)

"""Time k_enum on task ranges: python tools/slice_probe.py cfg4 lo:hi [lo:hi ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

n, s, d = G.make_config(sys.argv[1])
g = vdmc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
print("info", g.info, flush=True)
for spec in sys.argv[2:]:
    lo, hi = (int(x) for x in spec.split(":"))
    ts = []
    for _ in range(3):
        t = {}
        g.count(4, work=(lo, hi), timings=t)
        ts.append(t["enum"])
    print(f"{sys.argv[1]} tasks [{lo}, {hi}) enum best {min(ts):.2f} ms", flush=True)

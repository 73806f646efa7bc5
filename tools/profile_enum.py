"""Run one BASELINE config's count a few times (for ncu / quick timing):
python tools/profile_enum.py cfg3 4 [reps] [scale] [kind] [vertex|edges|layered]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
kind = sys.argv[5] if len(sys.argv) > 5 else "directed"
mode = sys.argv[6] if len(sys.argv) > 6 else "vertex"
n, s, d = G.make_config(name, scale=scale)
g = vdmc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
for _ in range(reps):
    t = {}
    if mode == "edges":
        out = g.count_edges(k, kind=kind, timings=t)
    else:
        out = g.count(k, kind=kind, timings=t, options={"layered": 1} if mode == "layered" else None)
    torch.cuda.synchronize()
tot = int(out.sum().item())
print(f"{name} k={k} {kind} {mode} enum_ms={t['enum']:.2f} schedule_ms={t['schedule']:.2f} "
      f"build_ms={g.info['build_ms']:.2f} sum={tot}" + ("" if mode == "edges" else f" sets={tot // k}"), flush=True)

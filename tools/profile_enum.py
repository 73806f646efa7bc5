"""Run one BASELINE config's count a few times (for ncu / quick timing):
python tools/profile_enum.py cfg3 4 [reps] [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

name, k = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
n, s, d = G.make_config(name, scale=scale)
g = vdmc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
g.set_profiling(True)
for _ in range(reps):
    out = g.count(k)
    torch.cuda.synchronize()
t = g.timings()
print(f"{name} k={k} enum_ms={t['enum']:.2f} plan_ms={t['plan']:.2f} build_ms={t['build']:.2f} "
      f"sets={int(out.sum().item()) // k}", flush=True)

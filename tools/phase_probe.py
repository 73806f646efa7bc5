"""Time k_enum with phases / loop kinds switched off (profiling only, results incomplete):
python tools/phase_probe.py cfg4 [k] [quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

name = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n, s, d = G.make_config(name)
g = vdmc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
g.set_profiling(True)
variants = [("full", {}), ("heavy only", {"VDMC_PHASES": "1"}), ("light only", {"VDMC_PHASES": "2"}),
            ("skip star3_heavy", {"VDMC_SKIP": "1"}), ("skip b in R", {"VDMC_SKIP": "2"}),
            ("skip b in L_a", {"VDMC_SKIP": "4"}), ("heavy, skip star", {"VDMC_PHASES": "1", "VDMC_SKIP": "1"}),
            ("heavy, skip b in R", {"VDMC_PHASES": "1", "VDMC_SKIP": "2"}),
            ("heavy, skip b in L_a", {"VDMC_PHASES": "1", "VDMC_SKIP": "4"}),
            ("heavy, skip all", {"VDMC_PHASES": "1", "VDMC_SKIP": "7"}),
            ("no cross items (fallback)", {"VDMC_SKIP": "8"}),
            ("heavy, skip all, no ca_build", {"VDMC_PHASES": "1", "VDMC_SKIP": "15"}),
            ("xblock 256", {"VDMC_XBLOCK": "256"}),
            ("xblock 1023", {"VDMC_XBLOCK": "1023"}),
            ("star block 512", {"VDMC_FOLD": "512"}), ("star block 256", {"VDMC_FOLD": "256"}),
            ("star 512 xblock 256", {"VDMC_FOLD": "512", "VDMC_XBLOCK": "256"}),
            ("heavy, only tasks with >= 128 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "128"}),
            ("heavy, only tasks with < 128 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "-128"}),
            ("heavy, only tasks with >= 512 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "512"}),
            ("heavy, only tasks with < 512 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "-512"})]
if len(sys.argv) > 3 and sys.argv[3] == "quick":
    variants = variants[:3]
elif len(sys.argv) > 3 and sys.argv[3] == "tasks":
    variants = variants[:2] + [v for v in variants if "VDMC_MINREM" in v[1]]
for label, env in variants:
    for key in ("VDMC_PHASES", "VDMC_SKIP", "VDMC_XBLOCK", "VDMC_FOLD", "VDMC_MINREM"):
        os.environ.pop(key, None)
    os.environ.update(env)
    ts = []
    for _ in range(3):
        out = g.count(k)
        torch.cuda.synchronize()
        ts.append(g.timings()["enum"])
        del out
    print(f"{name} k={k} {label:24s} enum {min(ts):8.2f} ms", flush=True)

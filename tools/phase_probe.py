"""Time k_enum with phases / loop kinds switched off (profiling build libvdmc_prof.so only,
results incomplete):  python tools/phase_probe.py cfg4 [k] [quick|tasks]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_11655_b200 import build as B  # noqa: E402

if "VDMC_LIB" not in os.environ:   # the switches below exist only in the profiling build (A/B variants are one)
    os.environ["VDMC_LIB"] = B.build_profiling()
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

name = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n, s, d = G.make_config(name)
g = vdmc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
variants = [("full", {}), ("heavy only", {"VDMC_PHASES": "1"}), ("light only", {"VDMC_PHASES": "2"}),
            ("skip star3_heavy", {"VDMC_SKIP": "1"}), ("skip b in R", {"VDMC_SKIP": "2"}),
            ("skip b in L_a", {"VDMC_SKIP": "4"}), ("heavy, skip star", {"VDMC_PHASES": "1", "VDMC_SKIP": "1"}),
            ("heavy, skip b in R", {"VDMC_PHASES": "1", "VDMC_SKIP": "2"}),
            ("heavy, skip b in L_a", {"VDMC_PHASES": "1", "VDMC_SKIP": "4"}),
            ("heavy, skip all", {"VDMC_PHASES": "1", "VDMC_SKIP": "7"}),
            ("no cross items (fallback)", {"VDMC_SKIP": "8"}),
            ("heavy, skip all, no ca_build", {"VDMC_PHASES": "1", "VDMC_SKIP": "15"}),
            ("xblock 128", {"cross_block": 128}),
            ("xblock 1023", {"cross_block": 1023}),
            ("star block 512", {"star_block": 512}), ("star block 256", {"star_block": 256}),
            ("heavy, only tasks with >= 128 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "128"}),
            ("heavy, only tasks with < 128 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "-128"}),
            ("heavy, only tasks with >= 512 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "512"}),
            ("heavy, only tasks with < 512 left", {"VDMC_PHASES": "1", "VDMC_MINREM": "-512"})]
if len(sys.argv) > 3 and sys.argv[3] == "closed":   # the closed-form heavy path's item kinds
    variants = variants[:3] + [("heavy, skip star items", {"VDMC_PHASES": "1", "VDMC_SKIP": "1"}),
                               ("heavy, skip j items", {"VDMC_PHASES": "1", "VDMC_SKIP": "2"}),
                               ("heavy, skip u walks", {"VDMC_PHASES": "1", "VDMC_SKIP": "4"}),
                               ("heavy, skip all items", {"VDMC_PHASES": "1", "VDMC_SKIP": "7"}),
                               ("light, skip b-in-R walks", {"VDMC_PHASES": "2", "VDMC_SKIP": "2"}),
                               ("light, skip b-in-L_a walks", {"VDMC_PHASES": "2", "VDMC_SKIP": "4"})]
elif len(sys.argv) > 3 and sys.argv[3] == "quick":
    variants = variants[:3]
elif len(sys.argv) > 3 and sys.argv[3] == "tasks":
    variants = variants[:2] + [v for v in variants if "VDMC_MINREM" in v[1]]
for label, env in variants:
    for key in ("VDMC_PHASES", "VDMC_SKIP", "VDMC_MINREM"):
        os.environ.pop(key, None)
    opts = {key: v for key, v in env.items() if not key.startswith("VDMC_")}
    os.environ.update({key: v for key, v in env.items() if key.startswith("VDMC_")})
    ts = []
    for _ in range(3):
        t = {}
        out = g.count(k, options=opts, timings=t)
        ts.append(t["enum"])
        del out
    print(f"{name} k={k} {label:24s} enum {min(ts):8.2f} ms", flush=True)

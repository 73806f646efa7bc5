"""A/B of result-preserving count options on one workload (same library, same graph):
python tools/ab_options.py cfg4 '{}' '{"star_block": 1023}' ...   -> best-of-3 k_enum ms each,
and a bit-identity check of every variant's matrix against the first."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

name = sys.argv[1]
variants = [json.loads(x) for x in sys.argv[2:]] or [{}]
k = 4
n, s, d = G.make_config(name)
g = vdmc.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
ref = None
for rep in range(2):
    for v in variants:
        ts = []
        for _ in range(3):
            t = {}
            out = g.count(k, options=v, timings=t)
            ts.append(t["enum"])
        if ref is None:
            ref = out.clone()
        same = torch.equal(out, ref)
        print(f"{name} {json.dumps(v):40s} enum best {min(ts):8.2f} ms  (all {', '.join(f'{x:.1f}' for x in ts)})"
              f"  identical={same}", flush=True)
        del out

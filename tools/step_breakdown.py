"""Where a bench step's time goes: host wall clock around each public call (synchronised)
plus the library's own event timings.  python tools/step_breakdown.py cfg5 [k] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as G  # noqa: E402
from paper_2201_11655_b200 import vdmc  # noqa: E402

name = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n, s, d = G.make_config(name)
ds, dd = torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda()
for it in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = vdmc.Graph(n, ds, dd)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tm = {}
    out = g.count(k, timings=tm)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    g.close()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    del out
    print(f"{name} k={k} rep {it}: build {1e3*(t1-t0):.1f} ms (events {g.info['build_ms']:.1f}); count host-return "
          f"{1e3*(t2-t1):.1f} ms, done {1e3*(t3-t1):.1f} ms (schedule {tm['schedule']:.1f} enum {tm['enum']:.1f} "
          f"finalize {tm['finalize']:.1f}); close {1e3*(t4-t3):.1f} ms", flush=True)

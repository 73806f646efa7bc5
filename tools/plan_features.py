"""Per-task cost features of the S4 planner under the default order (degree descending, ties by
id), summed per phase / remaining-position bucket, for fitting k_cost's constants against phase
timings (tools/phase_probe.py).  python tools/plan_features.py cfg4 > profiles/..."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen as G  # noqa: E402

name = sys.argv[1]
n, s, d = G.make_config(name)
a = np.concatenate([s, d]).astype(np.int64)
b = np.concatenate([d, s]).astype(np.int64)
key = np.unique(a * n + b)
u, v = key // n, key % n
deg = np.bincount(u, minlength=n)
order = np.lexsort((np.arange(n), -deg))
rank = np.empty(n, np.int64)
rank[order] = np.arange(n)
ru, rv = rank[u], rank[v]
o = np.lexsort((rv, ru))
ru, rv = ru[o], rv[o]
degr = deg[order]                      # degree by rank
off = np.zeros(n + 1, np.int64)
np.add.at(off, ru + 1, 1)
off = np.cumsum(off)
fwd = rv > ru
# tasks: forward entries in CSR order = root-major
tr, ta = ru[fwd], rv[fwd]
tidx = np.nonzero(fwd)[0]
split = np.searchsorted(tidx, off[:-1])          # index into tasks of each root's first task
D = np.diff(np.concatenate([split, [tidx.size]]))
i = np.arange(tidx.size) - split[tr]
rem = D[tr] - i - 1
da = degr[ta]
S2 = np.zeros(n, np.int64)
np.add.at(S2, ru, degr[rv])                      # sum of neighbour degrees per vertex
# suffix sums of R's degrees after a
fdeg = degr[ta].astype(np.int64)
cs = np.cumsum(fdeg)
root_end = (split + D)[tr] - 1
suf = cs[root_end] - cs                          # sum over R[j], j > i
heavy = degr[tr] > 128
feat = {
    "ntasks": int(tidx.size), "nheavy": int(heavy.sum()),
    "heavy": {}, "light": {},
}
def sums(mask):
    return {"count": int(mask.sum()), "rem2": float((rem[mask].astype(np.float64) ** 2).sum()),
            "rem": float(rem[mask].sum()), "da": float(da[mask].sum()), "S2a": float(S2[ta[mask]].sum()),
            "Dda": float((D[tr[mask]] * da[mask]).astype(np.float64).sum()), "suf": float(suf[mask].sum()),
            "remda": float((rem[mask] * da[mask]).astype(np.float64).sum()),
            "da2": float((da[mask].astype(np.float64) ** 2).sum())}
for lab, m in (("all", heavy), ("rem<128", heavy & (rem < 128)), ("rem>=128", heavy & (rem >= 128)),
               ("rem<512", heavy & (rem < 512)), ("rem>=512", heavy & (rem >= 512))):
    feat["heavy"][lab] = sums(m)
feat["light"]["all"] = sums(~heavy)
print(json.dumps(feat, indent=1))

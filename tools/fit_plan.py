"""Fit the S4 planner cost model (enum.cu k_cost) to measured slice times: per-task features of
the default order summed over the slices of bench.py --virtual-parts runs (profiles/<tag>/vparts_*.json)
plus phase totals; non-negative least squares on relative error.  python tools/fit_plan.py"""
import json, sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import graphgen as G
from scipy.optimize import nnls

def task_features(name):
    n, s, d = G.make_config(name)
    a = np.concatenate([s, d]).astype(np.int64); b = np.concatenate([d, s]).astype(np.int64)
    key = np.unique(a * n + b); u, v = key // n, key % n
    deg = np.bincount(u, minlength=n)
    order = np.lexsort((np.arange(n), -deg)); rank = np.empty(n, np.int64); rank[order] = np.arange(n)
    ru, rv = rank[u], rank[v]; o = np.lexsort((rv, ru)); ru, rv = ru[o], rv[o]
    degr = deg[order].astype(np.float64)
    off = np.zeros(n + 1, np.int64); np.add.at(off, ru + 1, 1); off = np.cumsum(off)
    fwd = rv > ru; tr, ta = ru[fwd], rv[fwd]; tidx = np.nonzero(fwd)[0]
    split = np.searchsorted(tidx, off[:-1]); D = np.diff(np.concatenate([split, [tidx.size]]))
    i = np.arange(tidx.size) - split[tr]; rem = (D[tr] - i - 1).astype(np.float64)
    da = degr[ta]
    S2 = np.zeros(n, np.float64); np.add.at(S2, ru, degr[rv])
    cs = np.cumsum(da); root_end = (split + D)[tr] - 1; suf = cs[root_end] - cs
    gk = ru * n + rv   # sorted
    pos = np.searchsorted(gk, ta * n + tr, side='right')
    nla = (off[ta + 1] - pos).astype(np.float64)          # a's neighbours with rank > r
    avgb = S2[ta] / np.maximum(da, 1)
    heavy = degr[tr] > 128
    Dd = D[tr].astype(np.float64)
    h, l = heavy * 1.0, (~heavy) * 1.0
    F = np.stack([h, h * rem ** 2, h * nla * Dd, h * nla * avgb,
                  l, l * suf, l * nla * avgb, l * rem * nla, l * nla ** 2, l * rem ** 2], axis=1)
    return F
names = ["h_cnt", "h_rem2", "h_nlaD", "h_Lwalk", "l_cnt", "l_suf", "l_Lwalk", "l_remnla", "l_nla2", "l_rem2"]
rows, ys = [], []
for cfg in ("cfg4", "cfg5"):
    F = task_features(cfg)
    
    C = np.vstack([np.zeros((1, F.shape[1])), np.cumsum(F, axis=0)])
    for tag in ("r02b", "r02d"):
        dd = json.loads(open(f"profiles/{tag}/vparts_{cfg}.json").read().strip().splitlines()[-1])
        for (lo, hi), ms in zip(dd["slices"], dd["slice_enum_ms"]):
            rows.append(C[hi] - C[lo]); ys.append(ms)
    hmask = F[:, 0] > 0
    if cfg == "cfg4":
        rows.append(F[hmask].sum(0)); ys.append(331.6)
        rows.append(F[~hmask].sum(0)); ys.append(121.4)
    else:
        rows.append(F.sum(0)); ys.append(327.5)
A = np.array(rows); y = np.array(ys)
w = 1 / y   # relative error
scale = A.max(0); scale[scale == 0] = 1
coef, res = nnls((A / scale) * w[:, None], y * w)
coef = coef / scale
pred = A @ coef
for nm, c in zip(names, coef): print(f"{nm:8s} {c:.4g}")
print("rel err per row:", np.round((pred - y) / y, 3))


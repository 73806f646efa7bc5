"""Fit the S4 planner cost model (enum.cu k_cost) to measured slice times: per-task features of
the default order, summed over the slices of bench.py --virtual-parts runs (gpurun_out/<tag>/
vparts_<cfg>_<G>.json), plus the heavy / light phase totals; non-negative least squares on the
relative error, with one free intercept per slice (kernel launch + tail, the same for every slice
and so irrelevant to the balance).   python tools/fit_plan.py TAG [TAG ...]"""
import glob
import json
import os
import sys

import numpy as np
from scipy.optimize import nnls

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen as G  # noqa: E402

NAMES = ["h_cnt", "h_D", "h_nla", "h_s2a", "h_rem", "h_Dda", "w_cnt", "w_D", "w_rem", "w_s2a",
         "l_cnt", "l_D", "l_nla", "l_s2a", "l_item", "l_itemsuf"]


def task_features(name):
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
    degr = deg[order].astype(np.float64)
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, ru + 1, 1)
    off = np.cumsum(off)
    fwd = rv > ru
    tr, ta = ru[fwd], rv[fwd]
    tidx = np.nonzero(fwd)[0]
    split = np.searchsorted(tidx, off[:-1])
    D = np.diff(np.concatenate([split, [tidx.size]]))
    i = np.arange(tidx.size) - split[tr]
    rem = (D[tr] - i - 1).astype(np.float64)
    da = degr[ta]
    S2 = np.zeros(n, np.float64)
    np.add.at(S2, ru, degr[rv])
    cs = np.cumsum(da)
    root_end = (split + D)[tr] - 1
    suf = cs[root_end] - cs                              # sum of deg(R[j]) over j > i
    rootsum = cs[root_end] - cs + da + (cs - cs[split[tr]] + da[split[tr]] - da)  # whole root (all j)
    gk = ru * n + rv
    pos = np.searchsorted(gk, ta * n + tr, side='right')
    nla = (off[ta + 1] - pos).astype(np.float64)         # a's neighbours with rank > r
    heavy = degr[tr] > 128
    Dd = D[tr].astype(np.float64)
    warp = heavy & (da <= 256)                     # heavy tasks run one per warp (enum.cu kWL)
    cta = heavy & ~warp
    h, w, l = cta * 1.0, warp * 1.0, (~heavy) * 1.0
    item = (i % 8 == 0) * 1.0                      # light items: <= 8 tasks (kLightChunk)
    F = np.stack([h, h * Dd, h * nla, h * S2[ta], h * rem, h * Dd * da / 1e3, w, w * Dd, w * rem, w * S2[ta],
                  l, l * Dd, l * nla, l * S2[ta], l * item, l * item * (suf + da)], axis=1)
    return F, heavy


def cxx(coef):
    """k_cost constants: ms per unit -> integer units of 1e-12 ms"""
    return {nm: int(round(c * 1e12)) for nm, c in zip(NAMES, coef)}


def main():
    tags = sys.argv[1:] or ["vp1"]
    rows, ys, icpt = [], [], []
    for cfg in ("cfg4", "cfg5"):
        F, heavy = task_features(cfg)
        C = np.vstack([np.zeros((1, F.shape[1])), np.cumsum(F, axis=0)])
        for tag in tags:
            for f in sorted(glob.glob(f"gpurun_out/{tag}/vparts_{cfg}_*.json")):
                dd = json.loads(open(f).read().strip().splitlines()[-1])
                for (lo, hi), ms in zip(dd["slices"], dd["slice_enum_ms"]):
                    rows.append(C[hi] - C[lo]); ys.append(ms); icpt.append(1.0)
            ph = f"gpurun_out/{tag}/phases_{cfg}.txt"
            if os.path.exists(ph):
                for line in open(ph):
                    if "heavy only" in line:
                        rows.append(F[heavy].sum(0)); ys.append(float(line.split()[-2])); icpt.append(1.0)
                    if "light only" in line:
                        rows.append(F[~heavy].sum(0)); ys.append(float(line.split()[-2])); icpt.append(1.0)
    A = np.hstack([np.array(rows), np.array(icpt)[:, None]])
    y = np.array(ys)
    w = 1 / y
    scale = A.max(0)
    scale[scale == 0] = 1
    coef, _ = nnls((A / scale) * w[:, None], y * w)
    coef = coef / scale
    pred = A @ coef
    for nm, c in zip(NAMES + ["intercept"], coef):
        print(f"{nm:10s} {c:.4g}")
    print("rel err per row:", np.round((pred - y) / y, 3))
    print("ns per unit:", {nm: round(c * 1e6, 4) for nm, c in zip(NAMES, coef)})
    print("k_cost integer weights (1e-12 ms):", cxx(coef))


if __name__ == "__main__":
    main()

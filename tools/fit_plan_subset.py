"""NNLS fit of the S4 planner cost model on a subset of tools/fit_plan.py's features:
    python tools/fit_plan_subset.py gpurun_out/TAG FEATURE...   (profiles/r02n_planner_fit.txt)"""
import sys, json, glob, os, numpy as np
from scipy.optimize import nnls
TAG=sys.argv[1]; ARGS=sys.argv[2:]; sys.path.insert(0,'tools'); sys.argv=['x']
import fit_plan as f
use = ARGS or None
rows, ys = [], []
for cfg in ('cfg4','cfg5'):
    F, heavy = f.task_features(cfg)
    C = np.vstack([np.zeros((1, F.shape[1])), np.cumsum(F, axis=0)])
    for fn in sorted(glob.glob(f'{TAG}/vparts_{cfg}_*.json')):
        d = json.loads(open(fn).read().strip().splitlines()[-1])
        for (lo, hi), ms in zip(d['slices'], d['slice_enum_ms']):
            rows.append(C[hi]-C[lo]); ys.append(ms)
    for line in open(f'{TAG}/phases_{cfg}.txt'):
        if 'heavy only' in line and cfg=='cfg4': rows.append(F[heavy].sum(0)); ys.append(float(line.split()[-2]))
        if 'light only' in line: rows.append(F[~heavy].sum(0)); ys.append(float(line.split()[-2]))
A=np.array(rows); y=np.array(ys)
sel=[f.NAMES.index(n) for n in (use or f.NAMES)]
A=A[:,sel]; names=[f.NAMES[i] for i in sel]
A=np.hstack([A, np.ones((len(y),1))])
w=1/y; sc=A.max(0); sc[sc==0]=1
coef,_=nnls((A/sc)*w[:,None], y*w); coef/=sc
pred=A@coef; err=(pred-y)/y
print('max|err| %.3f rms %.3f'%(abs(err).max(), np.sqrt((err**2).mean())))
print(np.round(err,2))
print({n: round(c*1e6,4) for n,c in zip(names+['icpt'],coef)})

"""Oracle study: do start-point features (attempts to factor H(x0), negative eigenvalues, pg, |f|, ...) predict which ncvx problems are expensive?  python scripts/order_predictors_ncvx.py"""
import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from oracle import pyoracle as po
from paper_2106_14995_b200 import synth
po.set_fast_forward(True)
def attempts(H):
    n=H.shape[0]; md=np.max(np.abs(np.diag(H))); a0=max(1e-3*md,1e-8); a=0.0
    for k in range(200):
        try:
            np.linalg.cholesky(H + a*np.eye(n)); return k
        except np.linalg.LinAlgError:
            a = max(2*a, a0)
    return 200
for d, N in ((8, 8192), (16, 4096), (4, 8192)):
    b = synth.ncvx(N, d)
    r = po.solve_batch(b, impl='oracle', workers=8)
    fl = r.flops.astype(float); ex=r.executed.astype(float); cg=r.cg_iterations.astype(float)
    x0 = np.clip(b.x0, b.lower, b.upper)
    F = np.zeros((N, 7))
    for i in range(N):
        f, g, H = po.family_eval(2, d, x0[i], b.params[i])
        Hs=0.5*(H+H.T); ev=np.linalg.eigvalsh(Hs)
        pg = g.copy(); pg[(x0[i] <= b.lower[i]) & (g > 0)] = 0; pg[(x0[i] >= b.upper[i]) & (g < 0)] = 0
        F[i]=[attempts(Hs), (ev<0).sum(), -ev.min()/max(np.abs(np.diag(H)).max(),1e-300), np.abs(pg).max(), abs(f), np.abs(b.params[i]).max(), np.linalg.norm(x0[i]-b.x0[i])]
    q=np.percentile(fl,90); heavy=fl>=q
    print(f"d={d}: flops p50 {np.median(fl):.0f} p90 {q:.0f} max {fl.max():.0f}; corr(flops, executed) {np.corrcoef(fl,ex)[0,1]:.2f} corr(flops, cg) {np.corrcoef(fl,cg)[0,1]:.2f}")
    for k,nm in enumerate(["attempts@x0","#neg eig","-eigmin/maxdiag","pg","|f|","max|prm|","|clip shift|"]):
        o=np.argsort(-F[:,k], kind='stable'); top=np.zeros(N,bool); top[o[:N//4]]=True
        sp = np.corrcoef(np.argsort(np.argsort(F[:,k])), np.argsort(np.argsort(fl)))[0,1]
        print(f"   {nm:16s}: heavy (top-10% flops) in top quarter {100*(heavy&top).sum()/heavy.sum():.0f}%  spearman {sp:.2f}")

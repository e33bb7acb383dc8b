"""Which d=2 cascade path flips zero/nonzero slack against the reference."""
import json, sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import golden
from paper_1804_03807_b200 import cascade, configs, rng as rngmod, tracker
from paper_1804_03807_b200.homotopy import TrackParams
from paper_1804_03807_b200.tracker import Solution
ch = golden("c3_cascade_chain")
pd = configs.c3()
d = int(sys.argv[1]) if len(sys.argv) > 1 else 2
emb = pd.emb.level(d)
X = ch[f"in{d}_x"]
h = cascade._slack_removal_homotopy(emb, rngmod.gamma_for(emb.seed, d))
res = tracker.track_batch(h, X)
nxt = emb.level(emb.k - 1)
sysn = nxt.system if nxt.k else nxt.base
rr = tracker.refine_batch(sysn, res.x[:, :-1][res.succeeded], tol=1e-13, max_iters=6, n_original=nxt.n_original)
n0 = pd.emb.n_original
refz = ch[f"out{d}_zero_x"]; refn = ch[f"out{d}_nonzero_x"]
ok = np.where(res.succeeded)[0]
for j, i in enumerate(ok):
    x = rr.x[j]
    sl = np.max(np.abs(x[n0:]))
    dz = np.min(np.max(np.abs(refz - x), axis=1)) if len(refz) else 9
    dn = np.min(np.max(np.abs(refn - x), axis=1)) if len(refn) else 9
    g_zero = rr.slack[j] == 4
    r_zero = dz < dn
    if g_zero != r_zero or min(dz, dn) > 1e-6:
        print(json.dumps({"path": int(i), "steps": int(res.steps[i]), "gpu_slack": float(sl), "gpu_zero": bool(g_zero),
                          "ref_zero": bool(r_zero), "d_to_ref_zero": float(dz), "d_to_ref_nonzero": float(dn),
                          "resid": float(rr.residual[j]), "cond": float(rr.condition[j]),
                          "ref_nonzero_slack_nearest": float(np.max(np.abs(refn[np.argmin(np.max(np.abs(refn - x), axis=1))][n0:]))) if len(refn) else None}))

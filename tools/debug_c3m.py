"""Dump the GPU C3-mini pipeline intermediates for offline comparison."""
import numpy as np
from paper_1804_03807_b200 import cascade, configs, filtering
pd = configs.c3_mini()
top, stats = cascade.solve_top(pd.emb, return_arrays=True)
sup = cascade.run_cascade(top, pd.emb)
out = {}
for lv in sup.levels:
    for kind, pts in (("zero", lv.zero_slack), ("nonzero", lv.nonzero_slack)):
        if pts:
            out[f"L{lv.dimension}_{kind}_x"] = np.array([s.coordinates for s in pts])
            out[f"L{lv.dimension}_{kind}_res"] = np.array([s.residual for s in pts])
            out[f"L{lv.dimension}_{kind}_cond"] = np.array([s.condition for s in pts])
wsets, stages = filtering.filter_junk(sup)
w = wsets[0]
n = pd.emb.n_original
cands = filtering._dedup(list(sup.levels[1].zero_slack), n)
Q = np.array([c.coordinates[:n] for c in cands])
v, _ = filtering.membership_batch(w, Q)
out["cand_q"] = Q
out["cand_v"] = v
out["W2"] = np.array([s.coordinates for s in w.points])
np.savez("gpurun_out/debug_c3m.npz", **out)
print("verdicts", v, [ (s.candidates, s.removed) for s in stages])

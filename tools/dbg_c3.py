import sys, os
sys.path.insert(0, ".")
import numpy as np
from paper_1804_03807_b200 import cascade, configs, tracker, systems
from paper_1804_03807_b200.homotopy import TrackParams
pd = configs.c3()
h, deg = cascade.top_homotopy(pd.emb)
system = pd.emb.system
X = np.random.default_rng(0).normal(size=(64, 14)) + 1j*np.random.default_rng(1).normal(size=(64, 14))
which = sys.argv[1]
if which == "refine":
    r = tracker.refine_batch(system, X, tol=1e-13, max_iters=2, n_original=8)
    print("refine ok", r.residual[:3])
elif which == "ddrefine":
    r = tracker.refine_dd_batch(system, X[:8], steps=2)
    print("ddrefine ok", r[1])
elif which == "track_nopolish":
    r = tracker.track_batch(h, None, TrackParams(dd_refine_singular=0), degrees=deg, count=256)
    print("track ok", r.counts())
elif which == "track":
    r = tracker.track_batch(h, None, TrackParams(), degrees=deg, count=256)
    print("track ok", r.counts(), r.counters)
elif which == "track_aux":
    st = systems.total_degree_starts(deg, 0, 64)
    r = tracker.track_batch(h, st, TrackParams(dd_refine_singular=0), trace=True)
    print("track aux ok", r.counts())
elif which == "track_explicit":
    st = systems.total_degree_starts(deg, 0, 64)
    r = tracker.track_batch(h, st, TrackParams(dd_refine_singular=0))
    print("track explicit ok", r.counts())

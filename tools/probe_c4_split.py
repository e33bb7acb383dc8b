"""C4 membership: kernel time split (track / endpoint) and host time."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1804_03807_b200 import _lib, cascade, configs, filtering  # noqa: E402

n_cand = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
pd = configs.c3()
top, st = cascade.solve_top(pd.emb, return_arrays=True)
lv = cascade._classify_level(top, pd.emb, pd.emb.k, cascade.TrackParams())
W = filtering.WitnessSet(pd.emb.k, pd.emb, lv.zero_slack)
cands, labels, info = configs.c4_candidates(pd, n_cand // 2, n_cand // 2, 44)
mh = filtering.MembershipHomotopy(W)
for rep in range(2):
    t0 = time.time()
    verdict, tracked = filtering.membership_batch(W, cands, mh=mh)
    dt = time.time() - t0
    c = _lib.last_counters()
    print(json.dumps({"candidates": len(cands), "paths": tracked, "wall_s": round(dt, 3),
                      "track_ms": round(c["kernel_ms_track"], 1), "endpoint_ms": round(c["kernel_ms_endpoint"], 1),
                      "dd_polished": c["dd_polished"], "evals_per_path": c["evals"] / tracked,
                      "agree": float(np.mean((verdict == 1) == (labels == 1)))}), flush=True)

"""C3 on the GPU, stage by stage: top continuation, then every cascade level
with its track/endpoint kernel times, evaluation counts and step statistics
(the per-level tail: a level lasts about as long as its slowest path)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, rng as rngmod  # noqa: E402
from paper_1804_03807_b200.homotopy import TrackParams  # noqa: E402
from paper_1804_03807_b200.tracker import track_batch  # noqa: E402

pd = configs.c3()
t0 = time.time()
top, st = cascade.solve_top(pd.emb, return_arrays=True)
c = top.counters
print(json.dumps({"stage": "top", "paths": len(top), "wall_s": round(time.time() - t0, 3),
                  "track_ms": c["kernel_ms_track"], "endpoint_ms": c["kernel_ms_endpoint"],
                  "steps_mean": float(top.steps.mean()), "steps_max": int(top.steps.max()),
                  "evals_per_path": c["evals"] / len(top)}), flush=True)
t1 = time.time()
lv = cascade._classify_level(top, pd.emb, pd.emb.k, TrackParams())
print(json.dumps({"stage": "classify top", "wall_s": round(time.time() - t1, 3), "counts": lv.counts}), flush=True)
tot = time.time()
while lv.dimension > 0:
    t1 = time.time()
    emb = lv.embedding
    h = cascade._slack_removal_homotopy(emb, rngmod.gamma_for(emb.seed, lv.dimension))
    starts = np.array([s.coordinates for s in lv.nonzero_slack])
    res = track_batch(h, starts, TrackParams())
    t2 = time.time()
    c = res.counters
    nxt = cascade._classify_arrays(res.x[:, :-1], res.succeeded, res.counts()["at_infinity"], res.counts()["failed"],
                                   emb.level(emb.k - 1), lv.dimension - 1, TrackParams(), len(res))
    t3 = time.time()
    st = np.sort(res.steps)
    print(json.dumps({"stage": f"level {lv.dimension}->{lv.dimension - 1}", "n": emb.nvars, "paths": len(res),
                      "track_wall_s": round(t2 - t1, 3), "track_ms": round(c["kernel_ms_track"], 1),
                      "endpoint_ms": round(c["kernel_ms_endpoint"], 1), "classify_wall_s": round(t3 - t2, 3),
                      "steps_mean": float(st.mean()), "steps_p99": int(st[int(0.99 * (len(st) - 1))]),
                      "steps_max": int(st[-1]), "evals_per_path": c["evals"] / len(res),
                      "dd_polished": c["dd_polished"], "counts": nxt.counts}), flush=True)
    lv = nxt
print(json.dumps({"stage": "cascade total", "wall_s": round(time.time() - tot, 3)}), flush=True)

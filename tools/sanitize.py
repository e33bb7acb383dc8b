"""Workload for compute-sanitizer (racecheck / memcheck / synccheck): a small
batch through every tracker kernel family and the endpoint / refine kernels.

    compute-sanitizer --tool racecheck python tools/sanitize.py
    compute-sanitizer --tool memcheck  python tools/sanitize.py

* parameter-bank kernel  track_pt_kernel<7>   : 96 C2 paths (device starts)
* table kernel (records) track_ctl_kernel<6>  : C3-mini top, 64 paths; <14>: 32 C3 top paths
* auxiliary kernel       track_aux_kernel<4>  : 8 C1 paths in double-double with traces
* endpoint_kernel (SVD + dd polish), refine_kernel, match_pairs_kernel
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, filtering, systems, tracker  # noqa: E402
from paper_1804_03807_b200.homotopy import LinearHomotopy, TrackParams  # noqa: E402

p2 = configs.c2()
r = tracker.track_batch(LinearHomotopy(p2.start, p2.target, p2.gamma), None, degrees=p2.degrees, count=96,
                        first_index=1000)
print("C2 96 paths:", r.counts(), flush=True)
pd = configs.c3_mini()
h, deg = cascade.top_homotopy(pd.emb)
r = tracker.track_batch(h, None, degrees=deg, count=64)
print("C3-mini top 64 paths:", r.counts(), flush=True)
lv = cascade._classify_level(r, pd.emb, pd.emb.k, TrackParams())
print("classify:", lv.counts, flush=True)
if lv.nonzero_slack:
    lv.nonzero_slack = lv.nonzero_slack[:16]
    print("cascade step:", cascade.cascade_step(lv).counts, flush=True)
pts = [s for s in lv.zero_slack + lv.nonzero_slack]
print("dedup:", len(filtering._dedup(pts, pd.emb.n_original)), "of", len(pts), flush=True)
p3 = configs.c3()
h3, deg3 = cascade.top_homotopy(p3.emb)
r = tracker.track_batch(h3, None, degrees=deg3, count=32, first_index=777)
print("C3 top 32 paths:", r.counts(), flush=True)
p1 = configs.c1()
st = systems.total_degree_starts(p1.degrees, 0, 8)
r = tracker.track_batch(LinearHomotopy(p1.start, p1.target, p1.gamma), st, TrackParams(precision="double_double"),
                        trace=True)
print("C1 dd 8 paths:", r.counts(), [len(t) for t in r.traces], flush=True)

"""Double-double tracking on a system with diverging paths, from the REFERENCE
(build container only; ~10 min): 16 paths of the C3-mini top continuation
(total-degree start, n = 6) with TrackParams(precision="double_double").  In
this mode there is no evaluation-noise floor (tracker.py:177-181, 461-477), so a
path whose coordinates grow cannot meet the fixed corrector tolerance and ends
FAILED where double precision classifies it at infinity.
    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_dd_c3m.py
-> tests/golden/track_c3m_dd.npz (also the double-precision statuses of the same paths)
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import nidpipe.tracker as rt  # noqa: E402

from make_golden import pack_results, ref_sys, save  # noqa: E402
from paper_1804_03807_b200 import cascade, configs, systems  # noqa: E402

pd = configs.c3_mini()
h, deg = cascade.top_homotopy(pd.emb)
idx = np.sort(np.random.default_rng(14).choice(int(np.prod(deg)), 16, replace=False))
starts = systems.total_degree_starts_at(deg, idx)
rh = rt.LinearHomotopy(ref_sys(h.start), ref_sys(h.target), h.gamma)
out = {"index": idx, "starts": starts}
for name, prm in (("double", rt.TrackParams()), ("dd", rt.TrackParams(precision="double_double"))):
    t0 = time.time()
    res = [rt.track(rh, x0, prm) for x0 in starts]
    print(name, [r.status for r in res], f"{time.time() - t0:.0f}s", flush=True)
    out.update({f"{name}_{k}": v for k, v in pack_results(res, h.dim).items()})
save("track_c3m_dd", **out)

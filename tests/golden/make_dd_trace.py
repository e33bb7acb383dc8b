"""Golden fixtures for the double-double tracking mode and the trace hook,
from the REFERENCE itself (build container only):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_dd_trace.py

* track_c1_dd.npz: all 16 C1 paths with TrackParams(precision="double_double")
  (`_track_dd`, tracker.py:461-497) and a 12-path C2 sample likewise, plus the
  reference's own small dd test system (tests/test_tracker.py:176-183).
* trace_c1.npz: the (t, step, corrector_iterations) traces of all 16 C1 paths
  and 24 C2 paths in double precision, and of the C1 paths in double-double
  (tracker.py:393-394).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

import nidpipe.tracker as rt  # noqa: E402

from make_golden import pack_results, ref_sys, save  # noqa: E402
from paper_1804_03807_b200 import configs, systems  # noqa: E402


def run(prob, index, params, with_trace):
    h = rt.LinearHomotopy(ref_sys(prob.start), ref_sys(prob.target), prob.gamma)
    starts = np.concatenate([systems.total_degree_starts(prob.degrees, int(i), 1) for i in index])
    res, traces = [], []
    t0 = time.time()
    for x0 in starts:
        tr = [] if with_trace else None
        res.append(rt.track(h, x0, params, tr))
        traces.append(tr)
    print(f"{prob.name}: {len(index)} paths ({params.precision}) in {time.time() - t0:.1f}s", flush=True)
    out = dict(index=np.asarray(index), starts=starts, **pack_results(res, prob.n))
    if with_trace:
        cap = max(len(t) for t in traces)
        tr = np.zeros((len(traces), cap, 3))
        for i, t in enumerate(traces):
            tr[i, :len(t)] = np.array(t).reshape(-1, 3)
        out["trace"] = tr
        out["trace_n"] = np.array([len(t) for t in traces], np.int32)
    return out


if __name__ == "__main__":
    c1, c2 = configs.c1(), configs.c2()
    dd = rt.TrackParams(precision="double_double")
    idx2 = np.sort(np.random.default_rng(11).choice(c2.paths, 24, replace=False))
    tr = {}
    tr.update({"c1_" + k: v for k, v in run(c1, np.arange(c1.paths), rt.TrackParams(), True).items()})
    tr.update({"c2_" + k: v for k, v in run(c2, idx2, rt.TrackParams(), True).items()})
    d1 = run(c1, np.arange(c1.paths), dd, True)
    tr.update({"c1dd_" + k: v for k, v in d1.items() if k.startswith("trace")})
    save("trace_c1", **tr)
    out = {"c1_" + k: v for k, v in d1.items() if not k.startswith("trace")}
    out.update({"c2_" + k: v for k, v in run(c2, idx2[:12], dd, False).items()})
    save("track_c1_dd", **out)

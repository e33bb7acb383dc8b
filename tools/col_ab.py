"""A/B of the column-owner evaluator (csrc/track_col.cuh) against the
row-per-warp records (NID_NO_COL=1) on a slice of the C3 top level.

    python tools/col_ab.py [P]"""
import json
import os
import subprocess
import sys

import numpy as np

P = int(sys.argv[1]) if len(sys.argv) > 1 else 18944
CHILD = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, flops, tracker
P = int(sys.argv[1])
pd = configs.c3()
h, degrees = cascade.top_homotopy(pd.emb, None)
fm = flops.flop_model(h.lowered())
for rep in range(2):
    r = tracker.track_batch(h, None, degrees=degrees, count=P, first_index=0)
    c = r.counters
    fl = fm.total(c["evals"], c["jacs"], c["scales"])
    print(json.dumps({"P": P, "counts": r.counts(), "kernel_ms": c["kernel_ms_track"],
                      "tflops": fl / (c["kernel_ms_track"] / 1e3) / 1e12, "evals_per_path": c["evals"] / P}), flush=True)
np.savez(sys.argv[2], status=r.status, x=r.x, steps=r.steps)
"""
out = {}
for name, env in (("rows", {"NID_NO_COL": "1"}), ("cols", {})):
    e = dict(os.environ)
    e.update(env)
    f = f"/tmp/col_ab_{name}.npz"
    print("==", name, flush=True)
    subprocess.run([sys.executable, "-c", CHILD, str(P), f], env=e, check=True)
    out[name] = np.load(f)
a, b = out["rows"], out["cols"]
same = a["status"] == b["status"]
fin = same & np.isin(a["status"], (0, 2))
dx = np.abs(a["x"][fin] - b["x"][fin]).max(axis=1) / np.maximum(1.0, np.abs(a["x"][fin]).max(axis=1)) if fin.any() else np.zeros(0)
print(json.dumps({"paths": int(P), "status_equal": int(same.sum()), "finite_both": int(fin.sum()),
                  "max_rel_endpoint_diff": float(dx.max()) if dx.size else None,
                  "steps_equal": int((a["steps"] == b["steps"]).sum())}))

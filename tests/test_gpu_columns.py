"""Column-owner evaluator (csrc/track_col.cuh) against the row-per-warp
records (NID_NO_COL=1) on the same 2,048 paths of the C3 top level.  The two
evaluators associate the sums differently, so endpoints agree to rounding, not
bitwise.  Cascade levels (shared and blended rows) and membership launches
(per-path coefficients) run through the column evaluator in the
reference-pinned tests of test_gpu_c3c4.py / test_gpu_fullsize.py."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1804_03807_b200 import cascade, configs, filtering, tracker
from paper_1804_03807_b200.homotopy import TrackParams
pd = configs.c3()
out = {}
# top level: 2,048 total-degree paths
h, degrees = cascade.top_homotopy(pd.emb, None)
r = tracker.track_batch(h, None, degrees=degrees, count=2048, first_index=12345)
out["top_status"], out["top_x"] = r.status, r.x
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, name, env):
    e = dict(os.environ)
    e.update(env)
    f = str(tmp_path / f"{name}.npz")
    subprocess.run([sys.executable, "-c", CHILD, ROOT, f], env=e, check=True, cwd=ROOT)
    return np.load(f)


def test_column_evaluator_matches_row_evaluator(nid, tmp_path):
    rows = _run(tmp_path, "rows", {"NID_NO_COL": "1"})
    cols = _run(tmp_path, "cols", {})
    same = rows["top_status"] == cols["top_status"]
    assert same.mean() >= 0.999, int((~same).sum())
    fin = same & np.isin(rows["top_status"], (0, 2))
    assert fin.sum() > 50
    d = np.abs(rows["top_x"][fin] - cols["top_x"][fin]).max(axis=1) / np.maximum(1.0, np.abs(rows["top_x"][fin]).max(axis=1))
    assert d.max() < 1e-9, float(d.max())

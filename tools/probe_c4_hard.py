"""C4 at full size (100,000 candidates): dump the candidates whose GPU verdict
differs from the construction label (plus a few agreeing controls) with the
GPU witness points, so the CPU oracle can decide them (tests/golden/make_c4_hard.py)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, filtering  # noqa: E402

pd = configs.c3()
top, st = cascade.solve_top(pd.emb, return_arrays=True)
lv = cascade._classify_level(top, pd.emb, pd.emb.k, cascade.TrackParams())
W = filtering.WitnessSet(pd.emb.k, pd.emb, lv.zero_slack)
cands, labels, info = configs.c4_candidates(pd, 50000, 50000, 44)
verdict, tracked = filtering.membership_batch(W, cands)
bad = np.where((verdict == 1) != (labels == 1))[0]
rng = np.random.default_rng(12)
ctrl = rng.choice(np.where((verdict == 1) == (labels == 1))[0], 6, replace=False)
sel = np.concatenate([bad, ctrl])
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/c4_hard.npz", index=sel, candidates=cands[sel], labels=labels[sel], gpu_verdict=verdict[sel],
         witness=np.array([s.coordinates for s in lv.zero_slack]))
print(json.dumps({"mismatch": bad.tolist(), "labels": labels[bad].tolist(), "verdicts": verdict[bad].tolist(),
                  "controls": ctrl.tolist()}))

"""Recipe for scratch/c5_cells.npz (build container only; needs the reference):

    PYTHONPATH=/root/reference/pkg/src python tools/make_c5_cells.py

The reference's lift_supports / enumerate_cells (polyhedral.py:67,597-621) on
C5's supports with seed 5 and solve_start_system's tie-retry loop
(cascade.py:124-149).  The output is ~1 MB and stays out of git (scratch/),
but travels to the GPU box with the snapshot for tools/probe_c5_polyhedral.py."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nidpipe.polyhedral as rph
from paper_1804_03807_b200 import configs, polyhedral as PH
p = configs.c5()
system = p.target
supports = PH.supports_of(system)
seed = 5
t0 = time.time()
for attempt in range(6):
    cells = []
    try:
        rph.enumerate_cells(rph.lift_supports(supports, seed, attempt), lambda c: cells.append(c) or True)
        break
    except rph.TieDetected:
        continue
print("cells", len(cells), "mv", sum(c.volume for c in cells), "attempt", attempt, "s", time.time() - t0, flush=True)
n = system.nvars
np.savez_compressed(os.path.join(ROOT, "scratch", "c5_cells.npz"),
                    pairs=np.array([[[a, b] for a, b in c.pairs] for c in cells], np.int8),
                    texps=np.array([np.concatenate([np.asarray(t, float) for t in c.texps]) for c in cells]),
                    volume=np.array([c.volume for c in cells], np.int32), seed=seed, attempt=attempt)
print("saved", flush=True)

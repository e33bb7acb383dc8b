"""C5 (cyclic support, n = 10) from the polyhedral start on the GPU, against
the total-degree start (bench.py's workload).

    python tools/probe_c5_polyhedral.py scratch/c5_cells.npz

The cells file comes from the reference's CPU LP (lift_supports /
enumerate_cells on C5's supports with seed 5; ~1,000 s in the build
container), saved by the recipe in DESIGN.md.  Prints: cells and mixed
volume; the start-system stage (all cells, one launch) and the g -> F
continuation (one launch); finite counts; and the cross-check that every
finite endpoint of the total-degree run appears among the polyhedral ones
(the reference's points_match, filtering.py:73-78, via the GPU all-pairs
matcher).
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1804_03807_b200 import configs, filtering, polyhedral as PH, rng as rngmod, tracker  # noqa: E402
from paper_1804_03807_b200.homotopy import LinearHomotopy  # noqa: E402


def main(path):
    d = np.load(path)
    p = configs.c5()
    system = p.target
    n = system.nvars
    supports = PH.supports_of(system)
    off = np.concatenate([[0], np.cumsum([len(s) for s in supports])])
    cells = [PH.Cell(tuple((tuple(map(int, pr[i, 0])), tuple(map(int, pr[i, 1]))) for i in range(n)),
                     tuple(tuple(tx[off[i]:off[i + 1]]) for i in range(n)), int(v))
             for pr, tx, v in zip(d["pairs"], d["texps"], d["volume"])]
    seed = int(d["seed"])
    g = PH.random_coefficient_system(supports, n, seed)
    out = {"cells": len(cells), "mixed_volume": int(d["volume"].sum())}
    PH.track_cells(cells[:4], g, supports)  # warm-up
    t0 = time.perf_counter()
    st, _ = PH.track_cells(cells, g, supports)
    out["start_s"] = time.perf_counter() - t0
    out["start_kernel_ms"] = st.counters["kernel_ms_track"]
    out["start_converged"] = int(st.succeeded.sum())
    x0 = st.x[st.succeeded]
    h = LinearHomotopy(g, system, rngmod.gamma_for(seed))
    t0 = time.perf_counter()
    res = tracker.track_batch(h, x0)
    out["continuation_s"] = time.perf_counter() - t0
    out["continuation_kernel_ms"] = res.counters["kernel_ms_track"]
    out["counts"] = res.counts()
    fin = res.x[res.status == 0]
    out["finite"] = int(len(fin))
    # total-degree run of bench.py's workload
    t0 = time.perf_counter()
    td = tracker.track_batch(LinearHomotopy(p.start, p.target, p.gamma), None, degrees=p.degrees,
                             count=int(np.prod(p.degrees)))
    out["total_degree_s"] = time.perf_counter() - t0
    tdf = td.x[td.status == 0]
    out["total_degree_finite"] = int(len(tdf))
    # every total-degree finite endpoint among the polyhedral ones (GPU all-pairs matcher)
    X = np.concatenate([fin, tdf])
    pairs = filtering.match_pairs(X)
    nf = len(fin)
    hit = np.zeros(len(tdf), bool)
    for a, b in pairs:
        a, b = int(a), int(b)
        if a < nf <= b:
            hit[b - nf] = True
        elif b < nf <= a:
            hit[a - nf] = True
    out["total_degree_found_in_polyhedral"] = int(hit.sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "scratch", "c5_cells.npz"))

"""Time the C2 polyhedral start system (115 cells, 924 paths) on the GPU:
one launch per cell (solve_cell) against every cell in one launch
(nid_track_cells).  Cells and g come from tests/golden/polyhedral_c2.npz.

    python tools/probe_polyhedral.py [reps]
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from test_polyhedral import load  # noqa: E402

from paper_1804_03807_b200 import polyhedral as PH  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    for name in ("c1", "c2"):
        g, gs, supports, cells = load(name)
        P = sum(c.volume for c in cells)
        PH.track_cells(cells, gs, supports)  # warm-up (module load, workspace)
        PH.solve_cell(cells[0], gs, supports)
        t0 = time.perf_counter()
        for _ in range(reps):
            for c in cells:
                PH.solve_cell(c, gs, supports)
        per_cell = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            res, _ = PH.track_cells(cells, gs, supports)
        batched = (time.perf_counter() - t0) / reps
        print(f"{name}: {len(cells)} cells, {P} paths, {int((res.status == 0).sum())} converged; "
              f"per-cell launches {per_cell * 1e3:.1f} ms ({P / per_cell:.0f} paths/s), "
              f"one launch {batched * 1e3:.1f} ms ({P / batched:.0f} paths/s; kernel "
              f"{res.counters.get('kernel_ms_track', float('nan')):.2f} ms), mean steps {np.mean(res.steps):.1f}")


def pipeline(lp_ms: float = 18.0):
    """C2 with a producer that pays lp_ms per cell (the reference's CPU LP
    enumerates C2's 115 cells in ~2.1 s, i.e. ~18 ms per cell): the
    pipeline's makespan against enumerate-all-then-track."""
    g, gs, supports, cells = load("c2")

    def producer():
        for c in cells:
            time.sleep(lp_ms * 1e-3)
            yield c

    t0 = time.perf_counter()
    allc = list(producer())
    PH.track_cells(allc, gs, supports)
    seq = time.perf_counter() - t0
    res, counts, st = PH.pipeline_cells(producer(), gs, supports)
    conv = sum(1 for r in res if r.status == "converged")
    print(f"c2 pipeline (LP {lp_ms} ms/cell): sequential {seq * 1e3:.0f} ms, pipelined {st.makespan * 1e3:.0f} ms "
          f"({st.batches} batches, consumer idle {st.consumer_idle * 1e3:.0f} ms, converged {conv}, "
          f"first consume before last produce: {st.first_consume_before_last_produce})")


if __name__ == "__main__":
    main()
    pipeline()

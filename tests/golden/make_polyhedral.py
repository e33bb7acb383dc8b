"""Golden fixtures for per-cell polyhedral tracking, made by running the
REFERENCE (nidpipe) itself.  Build container only:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_polyhedral.py

For the supports of C1 (dense quadrics, n = 4) and C2 (cyclic support,
n = 7): the reference's random-coefficient start system g
(`random_coefficient_system`, polyhedral.py:645-652), its lifting and
fine mixed cells (`lift_supports` / `enumerate_cells`, polyhedral.py:67,
597-621), and per cell the binomial start points and the tracked endpoints
of `solve_cell` (polyhedral.py:794-811).  Everything the GPU test needs is
stored as plain arrays; nothing here is read on the GPU box except the
committed .npz.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import nidpipe.polyhedral as rph  # noqa: E402
import nidpipe.tracker as rt  # noqa: E402
from nidpipe.parallel import work_crew  # noqa: E402

from make_golden import pack_results, ref_sys  # noqa: E402
from paper_1804_03807_b200 import configs  # noqa: E402

PROCS = int(os.environ.get("GOLDEN_PROCS", "8"))


def one(name, system, seed):
    supports = rph.supports_of(system)
    n = system.nvars
    g = rph.random_coefficient_system(supports, n, seed)
    cells = []
    for attempt in range(6):
        try:
            lifted = rph.lift_supports(supports, seed, attempt)
            rph.enumerate_cells(lifted, lambda c: cells.append(c) or True)
            break
        except rph.TieDetected:
            cells.clear()
    # g's terms in support order (PolyhedralHomotopy pairs them positionally)
    sup_flat, coef_flat, row_off = [], [], [0]
    for i, p in enumerate(g.polys):
        cmap = dict(p.terms)
        for e in supports[i]:
            sup_flat.append(e)
            coef_flat.append(cmap[e])
        row_off.append(len(sup_flat))
    out = dict(n=np.int32(n), seed=np.int64(seed), support=np.array(sup_flat, np.int32),
               coef=np.array(coef_flat, np.complex128), row_off=np.array(row_off, np.int32),
               ncells=np.int32(len(cells)))
    jobs = []
    for ci, cell in enumerate(cells):
        out[f"c{ci}_pairs"] = np.array([[a, b] for a, b in cell.pairs], np.int32)  # [n, 2, n]
        out[f"c{ci}_texps"] = np.concatenate([np.asarray(t, float) for t in cell.texps])
        out[f"c{ci}_volume"] = np.int32(cell.volume)
        coeff_of = [dict(p.terms) for p in g.polys]
        V = [[b[j] - a[j] for j in range(n)] for a, b in cell.pairs]
        beta = [-coeff_of[i][a] / coeff_of[i][b] for i, (a, b) in enumerate(cell.pairs)]
        starts = rph.binomial_solutions(V, beta)
        out[f"c{ci}_starts"] = np.array(starts)
        jobs.append(ci)
    t0 = time.time()
    res = work_crew(jobs, PROCS, lambda ci: rph.solve_cell(cells[ci], g, supports), mode="process")
    for ci, r in zip(jobs, res):
        for k, v in pack_results(r, n).items():
            out[f"c{ci}_{k}"] = v
    mv = sum(c.volume for c in cells)
    print(f"{name}: {len(cells)} cells, mixed volume {mv}, tracked in {time.time() - t0:.1f}s")
    np.savez_compressed(os.path.join(HERE, f"polyhedral_{name}.npz"), **out)


if __name__ == "__main__" and os.environ.get("POLY_CELLS", "1") == "1":
    one("c1", ref_sys(configs.c1().target), 11)
    one("c2", ref_sys(configs.c2().target), 12)


def top(name, pd):
    """The reference's solve_top with its default polyhedral start
    (cascade.py:214-246, solve_start_system :110-160) on an embedding: the
    cells it enumerated (cell_log), its start solutions and continuation
    results."""
    import nidpipe.cascade as rc

    from make_golden import ref_emb

    emb = ref_emb(pd.emb)
    log = []
    t0 = time.time()
    res, stats = rc.solve_top(emb, p=1, cell_log=log)
    print(f"{name}: {stats.cells} cells, mixed volume {stats.mixed_volume}, finite {stats.finite}, "
          f"at_inf {stats.at_infinity}, failures {stats.failures} in {time.time() - t0:.1f}s")
    n = emb.system.nvars
    out = dict(n=np.int32(n), ncells=np.int32(len(log)), cells=np.int32(stats.cells),
               mixed_volume=np.int64(stats.mixed_volume), start_failures=np.int32(stats.start_failures),
               finite=np.int32(stats.finite), at_infinity=np.int32(stats.at_infinity),
               failures=np.int32(stats.failures))
    for ci, cell in enumerate(log):
        out[f"c{ci}_pairs"] = np.array([[a, b] for a, b in cell.pairs], np.int32)
        out[f"c{ci}_texps"] = np.concatenate([np.asarray(t, float) for t in cell.texps])
        out[f"c{ci}_volume"] = np.int32(cell.volume)
    out.update({"top_" + k: v for k, v in pack_results(res, n).items()})
    np.savez_compressed(os.path.join(HERE, f"polyhedral_top_{name}.npz"), **out)


if __name__ == "__main__" and os.environ.get("POLY_TOP", "1") == "1":
    top("c3m", configs.c3_mini())


def decompose_golden(name, pd):
    """The reference's decompose (blackbox.py:36-110; polyhedral start,
    cascade, filter_junk, classify_isolated) on a base system: its cell log
    and the decomposition's counts."""
    import nidpipe.blackbox as rb

    f = ref_sys(pd.f)
    log = []
    t0 = time.time()
    rep = rb.decompose(f, top_dimension=pd.emb.k, seed=pd.seed, tasks=1, mode="thread", cell_log=log)
    print(f"{name} decompose: degrees {rep.degrees}, isolated {len(rep.isolated)}, suspects {len(rep.suspects)}, "
          f"cascade {rep.cascade_counts} in {time.time() - t0:.1f}s")
    n = pd.emb.system.nvars
    out = dict(n=np.int32(n), ncells=np.int32(len(log)),
               degrees=np.array(sorted(rep.degrees.items()), np.int64).reshape(-1, 2),
               isolated=np.array([s.coordinates for s in rep.isolated], np.complex128).reshape(-1, pd.f.nvars),
               suspects=np.int32(len(rep.suspects)),
               cascade=np.array([[c.get(k, 0) for k in ("dimension", "starts", "at_infinity", "zero_slack",
                                                         "nonzero_slack", "failures")] for c in rep.cascade_counts],
                                np.int64),
               stages=np.array([[s.candidate_dimension, s.against_dimension, s.candidates, s.removed]
                                for s in rep.filter_stages], np.int64).reshape(-1, 4))
    for ci, cell in enumerate(log):
        out[f"c{ci}_pairs"] = np.array([[a, b] for a, b in cell.pairs], np.int32)
        out[f"c{ci}_texps"] = np.concatenate([np.asarray(t, float) for t in cell.texps])
        out[f"c{ci}_volume"] = np.int32(cell.volume)
    np.savez_compressed(os.path.join(HERE, f"decompose_{name}.npz"), **out)
    # the reference's own deterministic JSON report of that run (report.py:81-128)
    import nidpipe.report as rr

    with open(os.path.join(HERE, f"report_{name}.json"), "w", encoding="utf-8") as fh:
        fh.write(rr.report_to_json(rep))
    with open(os.path.join(HERE, f"summary_{name}.txt"), "w", encoding="utf-8") as fh:
        fh.write(rr.summary_text(rep).split("timings:")[0])


if __name__ == "__main__" and os.environ.get("POLY_DECOMPOSE", "0") == "1":
    decompose_golden("c3m", configs.c3_mini())

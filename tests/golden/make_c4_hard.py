"""Golden verdicts for the hard C4 membership candidates, decided by the
REFERENCE itself (nidpipe.filtering.membership_test, filtering.py:92-127).

Input: gpurun_out/c4_hard.npz from tools/probe_c4_hard.py (a B200 run of the
full 100,000-candidate C4 batch): the candidates whose GPU verdict differs
from the construction label, six agreeing controls, and the GPU witness
points.  nidpipe decides each one from the same witness points; the verdicts
go to tests/golden/c4_hard.npz (`reference_verdict`), which
tests/test_gpu_c3c4.py compares the GPU against.  The CPU oracle's verdicts
(oracle/nid_oracle.py) are stored beside them (`oracle_verdict`) and
tests/test_oracle.py pins them equal.

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_c4_hard.py [--procs P]
"""
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def decide_reference(args):
    q, wit = args
    import nidpipe.filtering as rf
    import nidpipe.tracker as rt
    from make_golden import ref_emb
    from paper_1804_03807_b200 import configs

    pd = configs.c3()
    w = rf.WitnessSet(pd.emb.k, ref_emb(pd.emb), [rt.Solution(x, 0.0, 1.0) for x in wit])
    try:
        return 1 if rf.membership_test(w, q, 1, rt.TrackParams(), "thread") else 0
    except rf.MembershipIndeterminate:
        return -1


def decide_oracle(args):
    q, wit = args
    from oracle import nid_oracle as O
    from paper_1804_03807_b200 import configs

    pd = configs.c3()
    try:
        return 1 if O.membership_test(list(wit), pd.emb, q) else 0
    except O.MembershipIndeterminate:
        return -1


def main():
    procs = int(sys.argv[sys.argv.index("--procs") + 1]) if "--procs" in sys.argv else os.cpu_count()
    src = os.path.join(ROOT, "gpurun_out", "c4_hard.npz")
    if not os.path.exists(src):
        src = os.path.join(ROOT, "tests", "golden", "c4_hard.npz")
    d = np.load(src)
    jobs = [(q, d["witness"]) for q in d["candidates"]]
    with mp.get_context("spawn").Pool(min(procs, len(jobs))) as pool:
        ref_v = np.array(pool.map(decide_reference, jobs), dtype=np.int8)
        oracle_v = np.array(pool.map(decide_oracle, jobs), dtype=np.int8)
    gpu_v = d["gpu_verdict"] if "gpu_verdict" in d else d["gpu_verdict_r01"]
    np.savez(os.path.join(ROOT, "tests", "golden", "c4_hard.npz"), index=d["index"], candidates=d["candidates"],
             labels=d["labels"], witness=d["witness"], reference_verdict=ref_v, oracle_verdict=oracle_v,
             gpu_verdict_r01=gpu_v)
    print("reference", ref_v.tolist(), "oracle", oracle_v.tolist(), "gpu", gpu_v.tolist(), "labels",
          d["labels"].tolist())


if __name__ == "__main__":
    main()

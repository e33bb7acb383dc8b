"""Golden verdicts for the hard C4 membership candidates.

Input: gpurun_out/c4_hard.npz from tools/probe_c4_hard.py (a B200 run of the
full 100,000-candidate C4 batch): the candidates whose GPU verdict differs
from the construction label, six agreeing controls, and the GPU witness
points.  The CPU oracle (oracle/nid_oracle.py, the pinned restatement of
nidpipe.filtering.membership_test, filtering.py:92-127) decides each one from
the same witness points; the verdicts go to tests/golden/c4_hard.npz, which
tests/test_gpu_c3c4.py compares the GPU against.

    python tests/golden/make_c4_hard.py [--procs P]
"""
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def decide(args):
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
    d = np.load(os.path.join(ROOT, "gpurun_out", "c4_hard.npz"))
    jobs = [(q, d["witness"]) for q in d["candidates"]]
    with mp.get_context("spawn").Pool(min(procs, len(jobs))) as pool:
        oracle_v = np.array(pool.map(decide, jobs), dtype=np.int8)
    np.savez(os.path.join(ROOT, "tests", "golden", "c4_hard.npz"), index=d["index"], candidates=d["candidates"],
             labels=d["labels"], witness=d["witness"], oracle_verdict=oracle_v, gpu_verdict_r01=d["gpu_verdict"])
    print("oracle", oracle_v.tolist(), "gpu", d["gpu_verdict"].tolist(), "labels", d["labels"].tolist())


if __name__ == "__main__":
    main()

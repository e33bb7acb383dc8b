"""Time (and, under ncu, profile) a slice of the C3 top-level continuation
(n = 14, 4,068-term table: track_ctl_kernel<14>).

    python tools/probe_c3top.py [P] [first]"""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, flops, tracker  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
pd = configs.c3()
h, degrees = cascade.top_homotopy(pd.emb, None)
fm = flops.flop_model(h.lowered())
for rep in range(2):
    t0 = time.time()
    r = tracker.track_batch(h, None, degrees=degrees, count=P, first_index=first)
    dt = time.time() - t0
    c = r.counters
    fl = fm.total(c["evals"], c["jacs"], c["scales"])
    print(json.dumps({"P": P, "wall_s": dt, "counts": r.counts(), "kernel_ms": c["kernel_ms_track"],
                      "paths_per_s_kernel": P / (c["kernel_ms_track"] / 1e3),
                      "tflops": fl / (c["kernel_ms_track"] / 1e3) / 1e12,
                      "evals_per_path": c["evals"] / P}), flush=True)

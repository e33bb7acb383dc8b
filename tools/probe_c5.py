"""Time C5 subsets on the GPU and print per-launch counters."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_1804_03807_b200 import configs, tracker, flops
from paper_1804_03807_b200.homotopy import LinearHomotopy
p = configs.c5()
h = LinearHomotopy(p.start, p.target, p.gamma)
fm = flops.flop_model(h.lowered())
import paper_1804_03807_b200._lib as L
import ctypes as C
print("track regs n=10:", L.lib().nid_track_regs(10))
for P in [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [3000, 30000]:
    t0 = time.time()
    r = tracker.track_batch(h, None, degrees=p.degrees, count=P, first_index=0)
    dt = time.time() - t0
    c = r.counters
    fl = fm.total(c["evals"], c["jacs"], c["scales"])
    ph = (C.c_ulonglong * 7)()
    if hasattr(L.lib(), "nid_phase_cycles") and L.lib().nid_phase_cycles(ph) == 0 and sum(ph):
        names = ["control_top", "barrier_pre_eval", "eval", "barrier_post_eval", "ctl_after_eval", "lu", "backsub_ctl"]
        tot = sum(ph)
        print(json.dumps({k: round(v / tot, 4) for k, v in zip(names, ph)}))
    print(json.dumps({"P": P, "wall_s": dt, "paths_per_s": P / dt, "counts": r.counts(), "counters": c,
                      "tflops_track": fl / (c["kernel_ms_track"] / 1e3) / 1e12,
                      "steps_mean": float(r.steps.mean()), "steps_max": int(r.steps.max())}), flush=True)

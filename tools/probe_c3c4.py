"""C3 top continuation + cascade + filter on the GPU, and a C4 membership batch."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, filtering, tracker, systems
from paper_1804_03807_b200.homotopy import LinearHomotopy

pd = configs.c3()
t0 = time.time()
top, st = cascade.solve_top(pd.emb, return_arrays=True)
t1 = time.time()
print(json.dumps({"stage": "C3 top", "paths": len(top), "s": t1 - t0, "counts": top.counts(),
                  "counters": top.counters}), flush=True)
sup = cascade.run_cascade(top, pd.emb)
t2 = time.time()
print(json.dumps({"stage": "C3 cascade", "s": t2 - t1, "levels": sup.stage_counts}), flush=True)
if "--filter" in sys.argv:
    wsets, stages = filtering.filter_junk(sup)
    t3 = time.time()
    print(json.dumps({"stage": "C3 filter_junk", "s": t3 - t2, "witness": [(w.dimension, w.degree) for w in wsets],
                      "stages": [s.__dict__ for s in stages]}), flush=True)

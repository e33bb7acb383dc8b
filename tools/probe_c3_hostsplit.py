"""Where the C3 cascade's wall time goes, level by level: track launch
(C-ABI wall, kernel ms), refine launch, Python record building."""
import cProfile
import json
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs  # noqa: E402
from paper_1804_03807_b200.homotopy import TrackParams  # noqa: E402

pd = configs.c3()
top, st = cascade.solve_top(pd.emb, return_arrays=True)
lv = cascade._classify_level(top, pd.emb, pd.emb.k, TrackParams())
pr = cProfile.Profile()
t0 = time.time()
pr.enable()
levels = [lv]
while levels[-1].dimension > 0:
    levels.append(cascade.cascade_step(levels[-1]))
pr.disable()
print(json.dumps({"cascade_wall_s": round(time.time() - t0, 3), "levels": [l.counts for l in levels]}))
ps = pstats.Stats(pr)
ps.sort_stats("cumulative").print_stats(25)

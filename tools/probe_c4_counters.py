import sys, json, time
import numpy as np
sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, filtering, tracker
pd = configs.c3()
top, st = cascade.solve_top(pd.emb, return_arrays=True)
lv = cascade._classify_level(top, pd.emb, pd.emb.k, cascade.TrackParams())
W = filtering.WitnessSet(pd.emb.k, pd.emb, lv.zero_slack)
cands, labels, info = configs.c4_candidates(pd, 10000, 10000, 44)
from paper_1804_03807_b200 import _lib
t0 = time.time()
verdict, tracked = filtering.membership_batch(W, cands)
print(json.dumps({"tracked": tracked, "s": time.time() - t0, "counters": _lib.last_counters()}))

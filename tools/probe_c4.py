"""C4: witness set from the C3 top level, candidates, one membership launch."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
from paper_1804_03807_b200 import cascade, configs, filtering
from paper_1804_03807_b200.tracker import Solution

n_cand = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
pd = configs.c3()
t0 = time.time()
top, st = cascade.solve_top(pd.emb, return_arrays=True)
lv = cascade._classify_level(top, pd.emb, pd.emb.k, cascade.TrackParams())
W = filtering.WitnessSet(pd.emb.k, pd.emb, lv.zero_slack)
t1 = time.time()
print(json.dumps({"witness_degree": W.degree, "s": t1 - t0}), flush=True)
cands, labels, info = configs.c4_candidates(pd, n_cand // 2, n_cand // 2, 44)
t2 = time.time()
print(json.dumps({"candidates": len(cands), "s": t2 - t1, **info}), flush=True)
verdict, tracked = filtering.membership_batch(W, cands)
t3 = time.time()
agree = float(np.mean((verdict == 1) == (labels == 1)))
print(json.dumps({"membership_paths": tracked, "s": t3 - t2, "paths_per_s": tracked / (t3 - t2),
                  "agree_with_construction": agree, "indeterminate": int(np.sum(verdict < 0)),
                  "false_neg": int(np.sum((labels == 1) & (verdict != 1))),
                  "false_pos": int(np.sum((labels == 0) & (verdict == 1)))}), flush=True)

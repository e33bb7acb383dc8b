"""Per-shard kernel time of C5 split into W shards (strong-scaling balance):
contiguous index ranges, then strided shards (rank r: r, r+W, ...) as bench.py uses."""
import json, sys
sys.path.insert(0, ".")
from paper_1804_03807_b200 import configs, tracker
from paper_1804_03807_b200.homotopy import LinearHomotopy
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
p = configs.c5()
h = LinearHomotopy(p.start, p.target, p.gamma)
tracker.track_batch(h, None, degrees=p.degrees, count=20000, first_index=0)  # warm
P = p.paths
for mode in ("contiguous", "strided"):
    out = []
    for r in range(W):
        if mode == "contiguous":
            lo, cnt, st = r * P // W, (r + 1) * P // W - r * P // W, 1
        else:
            lo, cnt, st = r, (P - r + W - 1) // W, W
        res = tracker.track_batch(h, None, degrees=p.degrees, count=cnt, first_index=lo, index_stride=st)
        c = res.counters
        out.append({"mode": mode, "rank": r, "paths": cnt, "kernel_ms": round(c["kernel_ms_track"], 1),
                    "ep_ms": round(c["kernel_ms_endpoint"], 1), "evals_per_path": round(c["evals"] / cnt, 1)})
        print(json.dumps(out[-1]), flush=True)
    ks = [o["kernel_ms"] for o in out]
    print(json.dumps({"mode": mode, "W": W, "max_ms": max(ks), "mean_ms": sum(ks) / W,
                      "imbalance": max(ks) / (sum(ks) / W)}), flush=True)

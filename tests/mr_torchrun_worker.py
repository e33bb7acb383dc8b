"""Worker of tests/test_multirank.py::test_torchrun_two_ranks_gloo: launched by
`python -m torch.distributed.run --nproc-per-node 2` exactly as the driver
launches bench.py (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* from the
environment), on CPU with the gloo backend.  It runs the multi-rank plumbing
bench.py's native arm uses -- DistContext.from_env, the strided shard, the
finite-endpoint gather to rank 0, max / sum over ranks -- and the sharded
stage drivers, with the per-rank GPU call replaced by the CPU oracle (test
infrastructure).  Rank 0 prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from paper_1804_03807_b200 import configs, parallel, tracker  # noqa: E402
from paper_1804_03807_b200.homotopy import LinearHomotopy  # noqa: E402
from test_multirank import _patch  # noqa: E402

_patch()
ctx = parallel.DistContext.from_env(int(os.environ["WORLD_SIZE"]), backend="gloo")
p = configs.c2()
P = 48
lo, stride, Pl = ctx.shard_strided(P)
h = LinearHomotopy(p.start, p.target, p.gamma)
# the bench's shape: each rank tracks its own strided shard, endpoints gathered to rank 0
loc = tracker._track_local(h, None, degrees=p.degrees, count=Pl, first_index=lo, index_stride=stride)
x = torch.from_numpy(np.ascontiguousarray(loc.x).view(np.float64).reshape(Pl, p.n, 2))
got = parallel.gather_finite(ctx, x, torch.from_numpy(loc.status))
finite = ctx.sum_over_ranks(int(loc.succeeded.sum()))
slow = ctx.max_over_ranks(float(ctx.rank + 1))
# the stage-driver shape: every rank gets the whole batch back in job order
parallel.activate(ctx)
full = tracker.track_batch(h, None, degrees=p.degrees, count=P)
parallel.activate(None)
ctx.barrier()
if ctx.rank == 0:
    print(json.dumps({"world": ctx.world, "finite": finite, "gathered": int(got.shape[0]), "max": slow,
                      "full_finite": int(full.succeeded.sum()), "full_paths": len(full),
                      "status": full.status.tolist()}), flush=True)
ctx.close()

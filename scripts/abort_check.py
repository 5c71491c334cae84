#!/usr/bin/env python3
"""spd_context_abort on a two-GPU box (one process, one thread per GPU, the
drop-in's shape): rank 0 enters an SpMM whose boundary all-gather waits for
rank 1, rank 1 never joins; aborting rank 0's communicator must make its
call return an error instead of waiting forever.  Prints ABORT_RESULT."""
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import torch  # noqa: E402

from paper_2207_13901_b200 import _native as N  # noqa: E402
from paper_2207_13901_b200 import host as H  # noqa: E402

uid = H.Context.nccl_unique_id()
ctxs = [H.Context(d, use_torch_stream=False) for d in (0, 1)]
ths = [threading.Thread(target=ctxs[r].init_comm, args=(uid, r, 2)) for r in (0, 1)]
for t in ths:
    t.start()
for t in ths:
    t.join()
rng = np.random.default_rng(3)
n, m = 2000, 300
rows = rng.integers(0, n, 20000)
B = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, rng.integers(0, m, 20000)], 1),
                        rng.uniform(0.5, 1.5, 20000))
torch.cuda.set_device(0)
Bd = H.DeviceTensor.upload(ctxs[0], B)
Cd = torch.from_numpy(rng.uniform(size=m * 32)).cuda(0)
A = torch.zeros(n * 32, dtype=torch.float64, device="cuda:0")
H.partition_nonzero(ctxs[0], Bd, 1, 2)
res = {}


def rank0():
    try:
        H.spmm(ctxs[0], Bd, Cd, 32, A, first=0, count=1, pieces=2)  # stats: waits for the all-gather
        res["r"] = "returned"
    except Exception as ex:  # noqa: BLE001
        res["r"] = f"error: {type(ex).__name__}"


t = threading.Thread(target=rank0, daemon=True)
t.start()
time.sleep(3.0)
blocked = t.is_alive()
N.check(N.lib().spd_context_abort(ctxs[0].h))
t.join(timeout=30)
print("ABORT_RESULT", "PASS" if blocked and not t.is_alive() else "FAIL", "blocked_before_abort", blocked,
      "after", res.get("r"), flush=True)
os._exit(0)  # the aborted context is not torn down

#!/usr/bin/env python3
"""Device-side tensor construction on one B200.

COO -> CSR of the bench's R-MAT matrix (scale 24, 165.6 M distinct entries,
shuffled, plus 10% duplicate entries): spd_tensor_pack from device-resident
COO and from pinned host COO (H2D inside the timed region), checked against
the generator's CSR (rowptr/crd exact, vals within fp64 rounding of the
duplicate sums), beside the reference's own SparseTensor::pack
(oracle/_ref) timed on a bounded sample on the host.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402

import torch  # noqa: E402

from paper_2207_13901_b200 import host as H  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n, rp, crd, vals = bench.rmat_csr(scale, 10, 42)
rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
rng = np.random.default_rng(1)
perm = rng.permutation(crd.shape[0])
dup = rng.integers(0, crd.shape[0], crd.shape[0] // 10)
# duplicates split an entry's value in two: v = (v - 1) + 1 keeps the sum exact
r_all = np.concatenate([rows[perm], rows[dup]])
c_all = np.concatenate([crd[perm], crd[dup]])
v_main = vals[perm].copy()
v_dup = np.ones(dup.shape[0])
inv = np.empty_like(perm)
inv[perm] = np.arange(perm.shape[0])
np.subtract.at(v_main, inv[dup], 1.0)
v_all = np.concatenate([v_main, v_dup])
E = r_all.shape[0]
dev = torch.device("cuda", 0)
ctx = H.Context(0)
fmt = H.parse_format("ds")

rows_h = torch.from_numpy(r_all).pin_memory()
cols_h = torch.from_numpy(c_all).pin_memory()
vals_h = torch.from_numpy(v_all).pin_memory()
rows_d, cols_d, vals_d = rows_h.to(dev), cols_h.to(dev), vals_h.to(dev)


def timed(fn, reps=3):
    fn().close()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        t = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        t.close()
    return float(np.median(ts))


t_dev = timed(lambda: H.DeviceTensor.pack(ctx, (n, n), fmt, [rows_d, cols_d], vals_d))
t_host = timed(lambda: H.DeviceTensor.pack(ctx, (n, n), fmt, [rows_h.numpy(), cols_h.numpy()], vals_h.numpy()))
T = H.DeviceTensor.pack(ctx, (n, n), fmt, [rows_d, cols_d], vals_d)
got = T.download()
T.close()
ok_pattern = bool(np.array_equal(got.levels[1].rowptr(), rp) and np.array_equal(got.levels[1].crd, crd))
ok_vals = bool(np.all(np.abs(got.vals - vals) <= 1e-12 * np.maximum(np.abs(vals), 1.0)))

import oracle_bind as ob  # noqa: E402  (reference CPU pack: baseline only)

S = 1_000_000
t0 = time.perf_counter()
r = ob.RefRun.pack((n, n), "ds", np.stack([r_all[:S], c_all[:S]], axis=1), v_all[:S]).ok()
ref_s = r.exec_seconds()
print(json.dumps({
    "op": "pack COO->CSR (spd_tensor_pack)", "entries": int(E), "distinct": int(crd.shape[0]),
    "device_input_ms": t_dev * 1e3, "host_input_ms": t_host * 1e3,
    "device_mentries_per_s": E / t_dev / 1e6, "host_input_mentries_per_s": E / t_host / 1e6,
    "check_pattern_exact": ok_pattern, "check_vals": ok_vals,
    "reference_pack": {"entries": S, "seconds": ref_s, "mentries_per_s": S / ref_s / 1e6, "threads": 1,
                       "kind": "reference (oracle/_ref SparseTensor::pack)"},
}), flush=True)
ctx.close()

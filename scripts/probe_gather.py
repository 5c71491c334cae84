#!/usr/bin/env python3
"""Drives scripts/probe_gather.cu (measurement only): gather GB/s of 256-byte
row gathers vs gathers in flight / occupancy, for working sets in L2 and in
HBM, and for the R-MAT C2 column sequence itself."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

so = os.path.join(ROOT, "scripts", "libprobe_gather.so")
if not os.path.exists(so):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", so, os.path.join(ROOT, "scripts", "probe_gather.cu")], check=True)
lib = C.CDLL(so)
lib.probe_gather.restype = C.c_float
lib.probe_gather.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
NAMES = ["unr4_mb4", "unr8_mb4", "unr16_mb2", "unr4_mb6", "unr4_mb8", "unr8_mb6", "unr4_mb4_na", "unr8_mb4_na",
         "pipe4_mb4", "pipe8_mb3", "unr2_mb8", "unr16_mb3"]
dev = torch.device("cuda", 0)
n = 1 << 27
Crows = 1 << 24
Cd = torch.rand(Crows * 32, dtype=torch.float64, device=dev)
sink = torch.zeros(4, dtype=torch.float64, device=dev)
g = torch.Generator(device=dev)
g.manual_seed(1)
sets = {}
for mb in (16, 48, 2048, 4096):
    rows = min(Crows, mb * (1 << 20) // 256)
    sets[f"uniform_{mb}MB"] = torch.randint(0, rows, (n,), dtype=torch.int32, device=dev, generator=g)
if "--rmat" in sys.argv:
    import bench
    nn, rp, crd, vals = bench.rmat_csr(24, 10, 42)
    sets["rmat_c2_crd"] = torch.from_numpy(crd.astype("int32")).to(dev)
for name, idx in sets.items():
    m = idx.numel() - (idx.numel() % 32)
    for v, vn in enumerate(NAMES):
        grid = C.c_int()
        ms = lib.probe_gather(v, C.c_void_p(idx.data_ptr()), m, C.c_void_p(Cd.data_ptr()),
                              C.c_void_p(sink.data_ptr()), C.byref(grid))
        print(json.dumps({"set": name, "variant": vn, "grid": grid.value, "ms": round(ms, 4),
                          "gather_gbs": round(m * 256 / (ms * 1e-3) / 1e9, 1),
                          "mpos_per_ms": round(m / ms / 1e6, 2)}), flush=True)

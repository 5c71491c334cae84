#!/usr/bin/env python3
"""Drives scripts/probe_l2.cu: gather bandwidth of random 256-byte rows vs
the working-set size, for all SMs sharing the set (mode 0) and for SM
groups each reading half of it (modes 1 / 2).  DESIGN.md 7.1."""
import ctypes as C
import json
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = C.CDLL(os.path.join(HERE, "libprobe_l2.so"))
lib.probe_l2.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_int,
                         C.POINTER(C.c_float)]
buf = torch.rand(512 * 2**20 // 8, dtype=torch.float64, device="cuda")
sink = torch.zeros(1, dtype=torch.float64, device="cuda")
grid, per_warp = 148 * 8, 8192
rows_total = grid * 8 * per_warp
for mb in (16, 32, 48, 64, 80, 96, 112, 128, 160, 256, 512):
    nrows = mb * 2**20 // 256
    line = {"working_set_mb": mb}
    for mode, split in ((0, 0), (1, 74), (1, 70), (1, 78), (2, 0)):
        ms = C.c_float()
        rc = lib.probe_l2(buf.data_ptr(), nrows, per_warp, mode, split, sink.data_ptr(), grid, C.byref(ms))
        assert rc == 0, rc
        key = f"mode{mode}" + (f"_split{split}" if mode == 1 else "")
        line[key] = round(rows_total * 256 / ms.value / 1e6, 1)  # GB/s of gathered rows
    print(json.dumps(line), flush=True)

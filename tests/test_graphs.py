"""CUDA-graph replay of a step (spd_capture_begin/end, spd_graph_launch):
the replayed partition + leaf + combine gives bit-identical outputs to the
directly launched ops, for SpMV and SpMM over row and nonzero splits."""
import numpy as np
import pytest

import spd_kernels as K


@pytest.mark.gpu
@pytest.mark.parametrize("schedule", ["row", "nonzero"])
def test_graph_replay_matches_direct(schedule):
    import torch

    from paper_2207_13901_b200 import host as H

    stream = torch.cuda.Stream()
    ctx = H.Context(0, stream=stream.cuda_stream)
    rng = np.random.default_rng(31)
    n, m, N = 700, 500, 32
    rows = np.concatenate([np.full(5000, 3), rng.integers(0, n, 20000)])
    cols = rng.integers(0, m, rows.shape[0])
    B = H.SparseTensor.pack((n, m), H.parse_format("ds"), np.stack([rows, cols], 1), rng.uniform(0.5, 1.5, rows.shape[0]))
    Bd = H.DeviceTensor.upload(ctx, B)
    x = torch.from_numpy(rng.uniform(0.5, 1.5, m)).cuda()
    C = torch.from_numpy(rng.uniform(0.5, 1.5, m * N)).cuda()
    P = 5

    def step(y, A):
        if schedule == "row":
            H.partition_universe(ctx, Bd, P, host=False)
        else:
            H.partition_nonzero(ctx, Bd, 1, P, host=False)
        H.spmv(ctx, Bd, x, y, pieces=P, stats=False)
        H.spmm(ctx, Bd, C, N, A, pieces=P, stats=False)

    y0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    A0 = torch.zeros(n * N, dtype=torch.float64, device="cuda")
    with torch.cuda.stream(stream):
        step(y0, A0)  # direct (also builds the cached row views)
    stream.synchronize()
    y1 = torch.full((n,), 7.0, dtype=torch.float64, device="cuda")
    A1 = torch.full((n * N,), 7.0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    with ctx.capture() as cap:
        step(y1, A1)
    g = cap.graph
    for _ in range(3):
        g.launch()
    stream.synchronize()
    assert torch.equal(y0, y1) and torch.equal(A0, A1)
    g.close()
    # an op that reads back to the host cannot be captured
    with pytest.raises(Exception):
        with ctx.capture():
            H.partition_nonzero(ctx, Bd, 1, P, host=True)
    Bd.close()
    ctx.close()

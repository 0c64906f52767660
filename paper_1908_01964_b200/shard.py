"""Multi-GPU sharding of the hot path.

Every equation of the path is per frequency bin (and per utterance), so the
(utterance, bin) units split into contiguous, slot-balanced ranges with no
collective inside the EM loop; the only communication is the final gather of
the disjoint result slices to rank 0. One process per GPU (torch.distributed:
NCCL on B200, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, List, Tuple

import numpy as np


def partition(n_units: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous balanced ranges [lo, hi) of n_units over world ranks
    (sizes differ by at most one; empty ranges allowed when world > n_units)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    base, extra = divmod(max(n_units, 0), world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def shard_bins(inputs, params0, X, rank: int, world: int):
    """Slice RcscmInputs / RcscmParams / X (natural shapes) to this rank's bins."""
    lo, hi = partition(X.shape[0], world)[rank]
    sl = slice(lo, hi)
    inp = type(inputs)(inputs.a[sl], inputs.R_prime[sl], inputs.R_prime_pinv[sl], inputs.b[sl], inputs.n_h)
    p = type(params0)(params0.r_h[sl], params0.r_u[sl], params0.lam[sl])
    return (lo, hi), inp, p, X[sl]


def gather_params(local, rank: int, world: int, n_bins: int, J: int):
    """Gather each rank's (r_h, r_u, lam) slice to rank 0 -> full arrays on
    rank 0, None elsewhere. Uses torch.distributed point-to-point on CPU
    tensors (works with gloo; with NCCL pass device tensors instead)."""
    import torch
    import torch.distributed as dist

    parts = partition(n_bins, world)
    flat = np.concatenate([np.asarray(local.r_h, np.float64).ravel(), np.asarray(local.r_u, np.float64).ravel(),
                           np.asarray(local.lam, np.float64).ravel()])
    if rank != 0:
        if flat.size:
            dist.send(torch.from_numpy(flat), dst=0)
        return None
    r_h = np.zeros((n_bins, J))
    r_u = np.zeros((n_bins, J))
    lam = np.zeros(n_bins)
    for r, (lo, hi) in enumerate(parts):
        n = hi - lo
        if n == 0:
            continue
        if r == 0:
            buf = flat
        else:
            t = torch.empty(n * (2 * J + 1), dtype=torch.float64)
            dist.recv(t, src=r)
            buf = t.numpy()
        r_h[lo:hi] = buf[: n * J].reshape(n, J)
        r_u[lo:hi] = buf[n * J: 2 * n * J].reshape(n, J)
        lam[lo:hi] = buf[2 * n * J:]
    return r_h, r_u, lam


def solve_sharded(solve: Callable, inputs, params0, X, rank: int, world: int):
    """Run `solve(inputs, params0, X) -> params` on this rank's bins and gather
    the full (r_h, r_u, lam) on rank 0."""
    (_, _), inp, p, Xs = shard_bins(inputs, params0, X, rank, world)
    out = solve(inp, p, Xs) if Xs.shape[0] else type(params0)(np.zeros((0, X.shape[1])), np.zeros((0, X.shape[1])),
                                                              np.zeros(0))
    return gather_params(out, rank, world, X.shape[0], X.shape[1])

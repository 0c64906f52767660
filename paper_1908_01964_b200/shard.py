"""Multi-GPU sharding of the hot path.

Every equation of the path is per frequency bin (and per utterance), so the
(utterance, bin) units split into contiguous, slot-balanced ranges with no
collective inside the EM loop (the reference's bin partition is
parallel.hpp:50-80, called at solver_naive.hpp:429); the only communication is
the final gather of the disjoint result slices to rank 0. One process per GPU
(torch.distributed: NCCL with device tensors on B200, gloo with CPU tensors in
the CPU tests) -- the same functions serve both.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Tuple

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


def gather_rows(local, n_total: int, rank: int, world: int):
    """Gather each rank's contiguous row block (a torch tensor of shape
    (n_r, *rest), rows = this rank's partition(n_total, world) range) to rank 0
    with point-to-point sends -> the (n_total, *rest) tensor on rank 0 (same
    device and dtype as `local`), None elsewhere. NCCL needs device tensors,
    gloo CPU tensors; the blocks are disjoint, so the result does not depend on
    the rank count."""
    import torch
    import torch.distributed as dist

    parts = partition(n_total, world)
    rest = tuple(local.shape[1:])
    if rank != 0:
        if local.shape[0]:
            dist.send(local.contiguous(), dst=0)
        return None
    out = torch.empty((n_total,) + rest, dtype=local.dtype, device=local.device)
    for r, (lo, hi) in enumerate(parts):
        if hi == lo:
            continue
        if r == 0:
            out[lo:hi] = local
        else:
            dist.recv(out[lo:hi], src=r)
    return out


def gather_params(local, rank: int, world: int, n_bins: int, J: int, device: Optional[str] = None):
    """Gather each rank's (r_h, r_u, lam) bin slice to rank 0 -> full numpy
    arrays on rank 0, None elsewhere. device: where the transfer tensors live
    ("cuda:k" for NCCL, None / "cpu" for gloo)."""
    import torch

    dev = torch.device(device or "cpu")
    n = np.asarray(local.lam).shape[0]
    flat = np.concatenate([np.asarray(local.r_h, np.float64).reshape(n, J), np.asarray(local.r_u, np.float64).reshape(n, J),
                           np.asarray(local.lam, np.float64).reshape(n, 1)], axis=1)
    full = gather_rows(torch.from_numpy(flat).to(dev), n_bins, rank, world)
    if full is None:
        return None
    full = full.cpu().numpy()
    return full[:, :J].copy(), full[:, J:2 * J].copy(), full[:, 2 * J].copy()


def solve_sharded(solve: Callable, inputs, params0, X, rank: int, world: int, device: Optional[str] = None):
    """Run `solve(inputs, params0, X) -> params` on this rank's bins and gather
    the full (r_h, r_u, lam) on rank 0."""
    (_, _), inp, p, Xs = shard_bins(inputs, params0, X, rank, world)
    J = X.shape[1]
    out = solve(inp, p, Xs) if Xs.shape[0] else type(params0)(np.zeros((0, J)), np.zeros((0, J)), np.zeros(0))
    return gather_params(out, rank, world, X.shape[0], J, device)


class ShardedSession:
    """A batch of utterances strong-sharded over ranks: rank r keeps utterances
    partition(B, world)[r] resident in a device session (GpuContext.session_*),
    runs the pipeline stages on them with no communication, and gather() brings
    r_h, r_u, lambda and the Wiener dry output to rank 0 over the process
    group (NCCL device-to-device on GPUs).

    ctx: this rank's GpuContext; X, W, A, T, V: this rank's utterances only
    (the caller generates or loads just its range)."""

    def __init__(self, ctx, B_total: int, rank: int, world: int, X, W, A, T, V, n_h: int = 0):
        self.ctx, self.B, self.rank, self.world = ctx, B_total, rank, world
        self.lo, self.hi = partition(B_total, world)[rank]
        assert X.shape[0] == self.hi - self.lo, "X must hold exactly this rank's utterances"
        self.shape = X.shape
        ctx.session_load(X, W, A, T, V, n_h)

    def run(self, stages: int, iters: int = 0, hyper=None, eps_var: float = 1e-12):
        self.ctx.session_run(stages, iters, hyper, eps_var)

    def gather(self, device: str, want_dry: bool = True):
        """-> on rank 0 a dict of torch tensors r_h, r_u (B, I, J), lam (B, I)
        and dry (B, I, J) complex128 (device memory); None on other ranks. The
        session outputs are copied device-to-device into the transfer tensors
        (rcscm_gpu_session_fetch takes device pointers too), then gathered."""
        import torch

        n, I, J, _ = self.shape
        dev = torch.device(device)
        rh = torch.empty((n, I, J), dtype=torch.float64, device=dev)
        ru = torch.empty_like(rh)
        lam = torch.empty((n, I), dtype=torch.float64, device=dev)
        dry = torch.empty((n, I, J), dtype=torch.complex128, device=dev) if want_dry else None
        self.ctx.session_fetch_into(rh.data_ptr(), ru.data_ptr(), lam.data_ptr(),
                                    dry.data_ptr() if want_dry else 0)
        out = {"r_h": gather_rows(rh, self.B, self.rank, self.world),
               "r_u": gather_rows(ru, self.B, self.rank, self.world),
               "lam": gather_rows(lam, self.B, self.rank, self.world)}
        if want_dry:
            out["dry"] = gather_rows(torch.view_as_real(dry), self.B, self.rank, self.world)
        if self.rank != 0:
            return None
        if want_dry:
            out["dry"] = torch.view_as_complex(out["dry"])
        return out

"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded path: the
bin partition, per-rank solve and the final gather reproduce the unsharded
result bitwise (the per-bin arithmetic does not depend on the sharding)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1908_01964_b200.shard import partition


def test_partition_balanced():
    for n in (0, 1, 5, 513, 1025):
        for w in (1, 2, 3, 4, 8):
            parts = partition(n, w)
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path, backend):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_1908_01964_b200.shard import solve_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    inp, p, X = O.make_verify_instance(7, 24, 3, 77)
    res = solve_sharded(lambda i, q, x: O.run(backend, i, q, x, O.SolverOptions(iters=15)).params,
                        inp, p, X, rank, world)
    if rank == 0:
        np.savez(out_path, r_h=res[0], r_u=res[1], lam=res[2])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("backend", ["accel2", "naive"])
def test_sharded_equals_unsharded_gloo(O, tmp_path, backend):
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), out, backend), nprocs=2, join=True)
    got = np.load(out)
    inp, p, X = O.make_verify_instance(7, 24, 3, 77)
    ref = O.run(backend, inp, p, X, O.SolverOptions(iters=15)).params
    assert np.array_equal(got["r_h"], ref.r_h)
    assert np.array_equal(got["r_u"], ref.r_u)
    assert np.array_equal(got["lam"], ref.lam)


# ---- the GPU path as the per-rank solver (world_size 2, gloo transport) ----------
def _gpu_worker(rank, world, port, out_path, kind):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist

    from paper_1908_01964_b200 import GpuContext, Hyperparams, SolverOptions, synth
    from paper_1908_01964_b200.shard import ShardedSession, partition, solve_sharded
    import paper_1908_01964_b200._capi as C

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gpu = GpuContext(0)  # one GPU here: both ranks' kernels run on it, independently
    if kind == "bins":
        from oracle import oracle as O

        u = synth.make_config(1, utterances=1, I=37, J=640)[0]
        inp = O.build_noise_scm(u.W, u.A, u.X, 0)
        p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        res = solve_sharded(lambda i, q, x: gpu.run_algorithm2(i, q, Hyperparams(), x, SolverOptions(iters=25)).params,
                            inp, p0, u.X, rank, world)
        if rank == 0:
            np.savez(out_path, r_h=res[0], r_u=res[1], lam=res[2])
    else:  # utterances of a batched session (the bench's strong-scaling path)
        B = 5
        lo, hi = partition(B, world)[rank]
        X, W, A, T, V = synth.stack([synth.make_utterance(4, 24, 320, 0.05, 3000 + k) for k in range(lo, hi)])
        ss = ShardedSession(gpu, B, rank, world, X, W, A, T, V)
        ss.run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
        ss.run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 30)
        out = ss.gather("cpu")
        if rank == 0:
            np.savez(out_path, **{k: v.numpy() for k, v in out.items()})
    dist.barrier()
    gpu.close()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_bins_gpu_solver(O, gpu, tmp_path):
    """Bins of one utterance over 2 ranks, each solving its range with the CUDA
    path (run_algorithm2 through the C ABI), gathered to rank 0: bitwise equal
    to the single-process solve."""
    from paper_1908_01964_b200 import Hyperparams, SolverOptions, synth

    out = str(tmp_path / "bins.npz")
    mp.spawn(_gpu_worker, args=(2, _free_port(), out, "bins"), nprocs=2, join=True)
    got = np.load(out)
    u = synth.make_config(1, utterances=1, I=37, J=640)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    ref = gpu.run_algorithm2(inp, p0, Hyperparams(), u.X, SolverOptions(iters=25)).params
    assert np.array_equal(got["r_h"], ref.r_h)
    assert np.array_equal(got["r_u"], ref.r_u)
    assert np.array_equal(got["lam"], ref.lam)


@pytest.mark.gpu
def test_sharded_session_utterances(gpu, tmp_path):
    """The bench's multi-GPU path: 5 utterances over 2 ranks (3 + 2), each rank
    a device session running the fused solve + Wiener step, results gathered
    to rank 0 (ShardedSession.gather): bitwise equal to one session holding
    the whole batch."""
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    out = str(tmp_path / "utts.npz")
    mp.spawn(_gpu_worker, args=(2, _free_port(), out, "utts"), nprocs=2, join=True)
    got = np.load(out)
    X, W, A, T, V = synth.stack([synth.make_utterance(4, 24, 320, 0.05, 3000 + k) for k in range(5)])
    gpu.session_load(X, W, A, T, V, 0)
    gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 30)
    ref = gpu.session_fetch()
    for k in ("r_h", "r_u", "lam", "dry"):
        assert np.array_equal(got[k], ref[k]), k

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

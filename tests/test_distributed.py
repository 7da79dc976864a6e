"""Multi-GPU path: column sharding of Phi.

CPU (gloo, world size 2): the shard partition, the host plumbing of
paper_2105_10439_b200.distributed (NCCL-id broadcast, gathers) and the
sharded PCG decomposition (oracle/sharded.py restates the library's exchange
pattern) against the unsharded oracle.  GPU: the sharded entry point over a
real single-rank NCCL communicator reproduces the unsharded run bitwise.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cofem_oracle as O
from oracle.sharded import pcg_solve_sharded, pcg_solve_time_sharded
from paper_2105_10439_b200.distributed import column_shards, time_shards


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_column_shards_partition():
    for n_cols, world in [(65536, 8), (1000, 3), (16, 4), (1024, 1), (37, 2)]:
        shards = column_shards(n_cols, world)
        assert shards[0][0] == 0 and shards[-1][1] == n_cols
        for (a, b), (c, d) in zip(shards, shards[1:]):
            assert b == c
        for a, b in shards:
            assert a % 4 == 0 and b > a
        sizes = [b - a for a, b in shards]
        assert max(sizes) - min(sizes) <= 4
    with pytest.raises(ValueError):
        column_shards(4, 3)


def test_time_shards_geometry():
    from paper_2105_10439_b200.distributed import conv_halo

    assert time_shards(4096, 2, 256) == [(0, 2048), (2048, 4096)]
    s = time_shards(2**22, 8, 256)
    assert all(a % 256 == 0 for a, _ in s) and s[-1][1] == 2**22
    assert [b - a for a, b in s] == [2**19] * 8
    assert conv_halo(256) == 256 and conv_halo(257) == 256 and conv_halo(258) == 320 and conv_halo(1) == 0
    with pytest.raises(ValueError):
        time_shards(1024, 4, 513)  # 256-sample shards shorter than the 512-row halo
    with pytest.raises(ValueError):
        time_shards(512, 3, 2)  # fewer 256-sample units than ranks


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).copy())
        dist.all_reduce(t)
        return t.numpy()

    rng = np.random.default_rng(11)
    n, d, q = 48, 200, 7
    phi = (rng.standard_normal((n, d)) / np.sqrt(n)).astype(np.float32).astype(np.float64)
    alpha = rng.random(d) + 0.5
    B = rng.standard_normal((d, q))
    beta = 1e3
    minv = 1.0 / (beta + alpha)
    c0, c1 = column_shards(d, world)[rank]
    cfg = O.CgConfig(max_steps=300, tolerance=1e-10)
    rep = pcg_solve_sharded(phi[:, c0:c1], beta, alpha[c0:c1], B[c0:c1], minv[c0:c1], cfg, allreduce)
    parts = [None] * world
    dist.all_gather_object(parts, (c0, c1, rep.solution, rep.steps_taken, rep.final_relative_residual))

    # host plumbing of the product's distributed module: gather in rank order
    from paper_2105_10439_b200 import distributed as D

    sc = D.ShardedContext.__new__(D.ShardedContext)
    sc.world = world
    gathered = sc.gather(np.arange(c0, c1, dtype=np.float64))
    if rank == 0:
        np.save(out_path, np.concatenate([np.concatenate([p[2] for p in parts], axis=0).ravel(),
                                          [parts[0][3], parts[1][3], parts[0][4]],
                                          gathered]))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_pcg_matches_unsharded_oracle(tmp_path):
    out = str(tmp_path / "res.npy")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    res = np.load(out)
    rng = np.random.default_rng(11)
    n, d, q = 48, 200, 7
    phi = (rng.standard_normal((n, d)) / np.sqrt(n)).astype(np.float32).astype(np.float64)
    alpha = rng.random(d) + 0.5
    B = rng.standard_normal((d, q))
    beta = 1e3
    ref = O.pcg_solve(lambda V: O.system_apply(O.dense_op(phi), beta, alpha, V), B, 1.0 / (beta + alpha),
                      O.CgConfig(max_steps=300, tolerance=1e-10))
    X = res[: d * q].reshape(d, q)
    steps0, steps1, delta = res[d * q: d * q + 3]
    assert steps0 == steps1 == ref.steps_taken  # every rank takes the same decision
    assert np.linalg.norm(X - ref.solution) <= 1e-10 * np.linalg.norm(ref.solution)
    assert delta <= 1e-10 and ref.final_relative_residual <= 1e-10  # both converged; the last digits are rounding
    np.testing.assert_array_equal(res[d * q + 3:], np.arange(d))  # gather preserves rank order


def _conv_case():
    rng = np.random.default_rng(3)
    d, L, q = 1024, 90, 5
    h = np.exp(-np.arange(L) / 20.0)
    taps = h / np.linalg.norm(h)
    alpha = rng.random(d) + 0.5
    B = rng.standard_normal((d, q))
    beta = 400.0
    minv = 1.0 / (beta * O.conv_op(d, taps).col_sq_norms() + alpha)
    return d, taps, alpha, B, beta, minv


def _time_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    def allreduce(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).copy())
        dist.all_reduce(t)
        return t.numpy()

    def halo(rows, direction):
        """Send `rows` towards `direction`, receive the same-shaped block from the other side."""
        to, frm = rank + direction, rank - direction
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        recv = torch.zeros(rows.shape, dtype=torch.float64)
        reqs = []
        if 0 <= to < world:
            reqs.append(dist.isend(torch.from_numpy(rows.copy()), to))
        if 0 <= frm < world:
            reqs.append(dist.irecv(recv, frm))
        for r in reqs:
            r.wait()
        return recv.numpy()

    d, taps, alpha, B, beta, minv = _conv_case()
    t0, t1 = time_shards(d, world, taps.size)[rank]
    cfg = O.CgConfig(max_steps=300, tolerance=1e-10)
    rep = pcg_solve_time_sharded(taps, beta, alpha[t0:t1], B[t0:t1], minv[t0:t1], cfg, allreduce, halo)
    parts = [None] * world
    dist.all_gather_object(parts, (rep.solution, rep.steps_taken))
    if rank == 0:
        np.save(out_path, np.concatenate([np.concatenate([p[0] for p in parts], axis=0).ravel(),
                                          [p[1] for p in parts]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_time_sharded_convolution_pcg_matches_unsharded_oracle(tmp_path, world):
    """The convolution's time-shard decomposition (halo rows from the
    neighbours, scalars all-reduced) reproduces the unsharded float64 solve."""
    out = str(tmp_path / "res.npy")
    mp.start_processes(_time_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    res = np.load(out)
    d, taps, alpha, B, beta, minv = _conv_case()
    op = O.conv_op(d, taps)
    ref = O.pcg_solve(lambda V: beta * op.adjoint(op.apply(V)) + alpha[:, None] * V, B, minv,
                      O.CgConfig(max_steps=300, tolerance=1e-10))
    q = B.shape[1]
    X = res[: d * q].reshape(d, q)
    assert np.all(res[d * q:] == ref.steps_taken)
    assert np.linalg.norm(X - ref.solution) <= 1e-9 * np.linalg.norm(ref.solution)


@pytest.mark.gpu
def test_sharded_run_single_rank_nccl_matches_unsharded():
    """run_cofem_sharded over a real 1-rank NCCL communicator == run_cofem, bitwise."""
    from paper_2105_10439_b200 import _lib, run_cofem
    from paper_2105_10439_b200 import simulate as S
    from paper_2105_10439_b200.distributed import run_cofem_sharded

    if _lib.device_count() < 1:
        pytest.fail("needs a GPU")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        c = S.CONFIGS["dense-small"]
        prob, z, _ = S.dense_cs_problem(c)
        cfg = c.cofem_config("ozaki", iterations=5)
        st1, est1, d1 = run_cofem_sharded(prob, cfg)
        st2, est2, d2 = run_cofem(prob, cfg)
        np.testing.assert_array_equal(est1.mu, est2.mu)
        np.testing.assert_array_equal(st1.alpha, st2.alpha)
        assert [x["cg_steps"] for x in d1] == [x["cg_steps"] for x in d2]
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_time_sharded_convolution_single_rank_nccl_matches_unsharded():
    """The convolution through ShardedContext.for_operator / run_cofem_sharded
    over a real 1-rank NCCL communicator == run_cofem, bitwise."""
    from paper_2105_10439_b200 import _lib, run_cofem
    from paper_2105_10439_b200 import simulate as S
    from paper_2105_10439_b200.distributed import run_cofem_sharded

    if _lib.device_count() < 1:
        pytest.fail("needs a GPU")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        c = S.ConvConfig("conv-nccl", 4096, 256, 20.0, 0.01, 0.05, 10, 3, 200, 1e-5)
        prob, z = S.conv_problem(c)
        cfg = c.cofem_config("ozaki")
        st1, est1, d1 = run_cofem_sharded(prob, cfg)
        st2, est2, d2 = run_cofem(prob, cfg)
        np.testing.assert_array_equal(est1.mu, est2.mu)
        np.testing.assert_array_equal(st1.alpha, st2.alpha)
        assert [x["cg_steps"] for x in d1] == [x["cg_steps"] for x in d2]
    finally:
        dist.destroy_process_group()

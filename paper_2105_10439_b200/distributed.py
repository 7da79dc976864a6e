"""Column-sharded CoFEM across GPUs (one process per GPU).

Phi is split by columns (D) across ranks; each rank keeps its D_r columns,
all D-indexed vectors (alpha, mu, s, the PCG blocks) and its slice of the
probes.  Per PCG step the only exchanges are an NCCL all-reduce of the
N x (K+1) partial products Phi_r P_r and two small all-reduces of the
per-column PCG scalars -- issued by the native library on its own stream
(include/cofem_b200.h: cofem_set_comm).  torch.distributed is the plumbing
that launches the ranks and ships the 128-byte NCCL id.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .cofem import PROBE_STREAM, PrecisionState, PosteriorEstimate, _theta_args
from .problem import substream
from .cg import DivergenceError

ALIGN = 4  # shard boundaries on 4-column multiples (device RNG / vector loads)


def column_shards(n_cols, world_size, align=ALIGN):
    """Balanced [start, stop) column ranges, boundaries multiples of `align`."""
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    units = -(-n_cols // align)
    bounds = [min(n_cols, align * (units * r // world_size)) for r in range(world_size + 1)]
    bounds[-1] = n_cols
    shards = [(bounds[r], bounds[r + 1]) for r in range(world_size)]
    if any(b <= a for a, b in shards):
        raise ValueError(f"{n_cols} columns cannot be split across {world_size} ranks")
    return shards


def _dist():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("torch.distributed must be initialised (one process per GPU)")
    return dist


def broadcast_nccl_id(dist, rank, device):
    """Rank 0 creates the NCCL unique id; every rank receives it."""
    import torch

    uid = _lib.nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.to(f"cuda:{device}")
    dist.broadcast(t, src=0)
    return bytes(t.cpu().tolist())


class ShardedContext:
    """A rank's native context on its column shard, joined to the NCCL group."""

    def __init__(self, n_rows, n_cols, precision="fp32", device=0, phi=None, seed=None, scale=None):
        dist = _dist()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.shards = column_shards(n_cols, self.world)
        c0, c1 = self.shards[self.rank]
        self.col_range = (c0, c1)
        self.n_rows, self.n_cols = n_rows, n_cols
        code = {"fp32": _lib.FP32, "fp64": _lib.FP64, "ozaki": _lib.OZAKI}[precision]
        self.ctx = _lib.Context(n_rows, c1 - c0, code, device)
        self.ctx.set_shard(c0, n_cols)
        if phi is not None:
            self.ctx.set_dictionary(np.ascontiguousarray(phi[:, c0:c1]))
        elif seed is not None:
            self.ctx.generate_gaussian(seed, scale)
        uid = broadcast_nccl_id(dist, self.rank, device)
        self.ctx.set_comm(uid, self.world, self.rank)

    def gather(self, local):
        """Concatenate a D-indexed local vector across ranks (rank order)."""
        dist = _dist()
        parts = [None] * self.world
        dist.all_gather_object(parts, np.asarray(local))
        return np.concatenate(parts)


def run_cofem_sharded(problem, cfg, device=0, sharded=None):
    """run_cofem (cofem.py:136-157) with Phi column-sharded over the process group.

    Every rank passes the same host problem; each uploads only its columns.
    Returns the full (gathered) PrecisionState, PosteriorEstimate and
    diagnostics on every rank.
    """
    dim = problem.dim
    if sharded is None:
        sharded = ShardedContext(problem.op.n_rows, dim, cfg.cg.precision, device, phi=problem.op.matrix)
    c0, c1 = sharded.col_range
    theta_code, theta = _theta_args(cfg.cg.theta_policy, dim)
    # every rank draws its rows of the reference's probe stream on its device
    sharded.ctx.set_probe_stream(substream(cfg.seed, PROBE_STREAM))
    try:
        out, failure = sharded.ctx.run(problem.y, problem.beta, cfg.iterations, cfg.probes,
                                       _lib.VARIANT_CODES[cfg.variant], theta_code, cfg.clamp_max, cfg.floor_eps,
                                       cfg.cg.max_steps, cfg.cg.tolerance, cfg.cg.printed_recursion,
                                       None if theta is None else theta[c0:c1], None)
    finally:
        sharded.ctx.set_probe_stream(None)
    if failure is not None:
        it, step = failure
        raise DivergenceError(step, f"EM iteration {it}")
    alpha, mu, s, steps, resid = out
    alpha, mu, s = sharded.gather(alpha), sharded.gather(mu), sharded.gather(s)
    state = PrecisionState(alpha, cfg.iterations, cfg.clamp_max, cfg.floor_eps)
    diagnostics = [{"iteration": t + 1, "cg_steps": int(steps[t]), "cg_residual": float(resid[t])}
                   for t in range(cfg.iterations)]
    return state, PosteriorEstimate(mu, s, None), diagnostics

"""Sharded CoFEM across GPUs.

Dense dictionaries are split by columns (D) across ranks; each rank keeps its
D_r columns, all D-indexed vectors (alpha, mu, s, the PCG blocks) and its
slice of the probes.  Per PCG step the only exchanges are an all-reduce of
the N x (K+1) partial products Phi_r P_r and two small all-reduces of the
per-column PCG scalars.

Convolution dictionaries (BASELINE config 3) are split in time: rank r holds
samples [t_r, t_{r+1}) of both the signal and the observation (Phi is square
Toeplitz).  Phi P needs the previous shard's last L-1 samples of P and Phi^T V
the next shard's first L-1 samples of V, so per contraction the ranks agree
on the operand's int8 scales (an all-reduce(max) of QW column maxima) and
swap one halo of lpad rows of int8 digit planes with their neighbours; the
PCG scalars are all-reduced as for dense shards.  Nothing N x Q is reduced.

All exchanges are issued by the native library on its own stream.  Two
transports implement them (include/cofem_b200.h):
* an NCCL communicator, one process per GPU (``ShardedContext`` /
  ``run_cofem_sharded``; torch.distributed only ships the 128-byte NCCL id);
* an in-process shard group, one host thread per rank (``run_cofem_threaded``;
  ranks on one device or on peer-accessible devices).
"""

from __future__ import annotations

import threading

import numpy as np

from . import _lib
from .cg import DivergenceError
from .cofem import PROBE_STREAM, PosteriorEstimate, PrecisionState, _theta_args
from .operators import ConvolutionOperator, DenseOperator, PartialDct2Operator
from .problem import substream

ALIGN = 4  # dense shard boundaries on 4-column multiples (device RNG / vector loads)
TIME_ALIGN = 256  # convolution shard boundaries (the library's row padding)


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


def conv_halo(n_taps):
    """Halo rows a convolution shard exchanges: L-1 rounded up to 64."""
    return -(-(int(n_taps) - 1) // 64) * 64


def time_shards(n_samples, world_size, n_taps=1):
    """Balanced [start, stop) sample ranges of a time-sharded convolution:
    boundaries on 256-sample multiples, every shard but the last at least the
    filter halo long (the library exchanges halos with neighbours only)."""
    shards = column_shards(n_samples, world_size, TIME_ALIGN)
    halo = conv_halo(n_taps)
    for a, b in shards[:-1]:
        if b - a < halo:
            raise ValueError(f"{n_samples} samples over {world_size} ranks leave shards shorter than the "
                             f"{halo}-sample filter halo")
    return shards


def shard_ranges(op, world_size):
    if isinstance(op, ConvolutionOperator):
        return time_shards(op.n_cols, world_size, op.gpu_taps().size)
    if isinstance(op, PartialDct2Operator):
        raise NotImplementedError("2-D DCT dictionaries run on one GPU (their transposes are not sharded)")
    if isinstance(op, DenseOperator):
        return column_shards(op.n_cols, world_size)
    raise TypeError(f"cannot shard a {type(op).__name__}")


def shard_context(op, precision, device, c0, c1):
    """The native context of shard [c0, c1) of `op` (not yet joined to a
    transport; a dense shard's dictionary is uploaded by upload_shard once it
    has joined)."""
    precision = op.resolve_precision(precision)
    if isinstance(op, ConvolutionOperator):
        if precision not in ("ozaki", "ozaki24"):
            raise NotImplementedError("time-sharded convolutions run the 'ozaki' (int8 band) kernels")
        ctx = _lib.Context.convolution(c1 - c0, op.gpu_taps(), _lib.OZAKI24 if precision == "ozaki24" else _lib.OZAKI,
                                       device)
    else:
        code = {"fp32": _lib.FP32, "fp64": _lib.FP64, "ozaki": _lib.OZAKI, "ozaki24": _lib.OZAKI24}[precision]
        ctx = _lib.Context(op.n_rows, c1 - c0, code, device)
    ctx.set_shard(c0, op.n_cols)
    return ctx


def upload_shard(ctx, op, c0, c1):
    """Upload a dense shard's columns after the context joined its transport:
    a float64 dictionary goes up exactly (the fp64 mode multiplies it, the
    ozaki planes are built from it -- collectively, with the row scales
    shared across the ranks, so every rank calls this together)."""
    if not isinstance(op, DenseOperator):
        return
    cols = np.ascontiguousarray(op.matrix[:, c0:c1])
    if cols.dtype == np.float64:
        ctx.set_dictionary_f64(cols)
    else:
        ctx.set_dictionary(cols)


def local_observation(op, y, c0, c1):
    """The rows of y a shard consumes: all of them (dense), its samples (convolution)."""
    return np.asarray(y)[c0:c1] if isinstance(op, ConvolutionOperator) else np.asarray(y)


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
    """A rank's native context on its shard, joined to the NCCL group.

    ``ShardedContext(n_rows, n_cols, ...)`` builds a dense column shard (from
    a host ``phi`` or the device generator); ``ShardedContext.for_operator``
    shards a DenseOperator by columns or a ConvolutionOperator in time."""

    def __init__(self, n_rows, n_cols, precision="fp32", device=0, phi=None, seed=None, scale=None, _op=None):
        dist = _dist()
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        if _op is not None:
            self.shards = shard_ranges(_op, self.world)
            c0, c1 = self.shards[self.rank]
            self.ctx = shard_context(_op, precision, device, c0, c1)
        else:
            self.shards = column_shards(n_cols, self.world)
            c0, c1 = self.shards[self.rank]
            if precision == "auto":
                precision = "ozaki24"  # a dictionary worth sharding is large
            code = {"fp32": _lib.FP32, "fp64": _lib.FP64, "ozaki": _lib.OZAKI, "ozaki24": _lib.OZAKI24}[precision]
            self.ctx = _lib.Context(n_rows, c1 - c0, code, device)
            self.ctx.set_shard(c0, n_cols)
            if phi is not None:
                self.ctx.set_dictionary(np.ascontiguousarray(phi[:, c0:c1]))
            elif seed is not None:
                self.ctx.generate_gaussian(seed, scale)
        self.col_range = (c0, c1)
        self.n_rows, self.n_cols = n_rows, n_cols
        uid = broadcast_nccl_id(dist, self.rank, device)
        self.ctx.set_comm(uid, self.world, self.rank)
        if _op is not None:
            upload_shard(self.ctx, _op, c0, c1)

    @classmethod
    def for_operator(cls, op, precision="ozaki", device=0):
        return cls(op.n_rows, op.n_cols, precision, device, _op=op)

    def gather(self, local):
        """Concatenate a D-indexed local vector across ranks (rank order)."""
        dist = _dist()
        parts = [None] * self.world
        dist.all_gather_object(parts, np.asarray(local))
        return np.concatenate(parts)


def _run_shard(ctx, problem, cfg, c0, c1):
    """One rank's cofem_run on its shard; returns (alpha, mu, s, steps, resid)."""
    theta_code, theta = _theta_args(cfg.cg.theta_policy, problem.dim)
    # every rank draws its rows of the reference's probe stream on its device
    ctx.set_probe_stream(substream(cfg.seed, PROBE_STREAM))
    try:
        out, failure = ctx.run(local_observation(problem.op, problem.y, c0, c1), problem.beta, cfg.iterations,
                               cfg.probes, _lib.VARIANT_CODES[cfg.variant], theta_code, cfg.clamp_max,
                               cfg.floor_eps, cfg.cg.max_steps, cfg.cg.tolerance, cfg.cg.printed_recursion,
                               None if theta is None else theta[c0:c1], None)
    finally:
        ctx.set_probe_stream(None)
    if failure is not None:
        it, step = failure
        raise DivergenceError(step, f"EM iteration {it}")
    return out


def _assemble(cfg, alpha, mu, s, steps, resid):
    state = PrecisionState(alpha, cfg.iterations, cfg.clamp_max, cfg.floor_eps)
    diagnostics = [{"iteration": t + 1, "cg_steps": int(steps[t]), "cg_residual": float(resid[t])}
                   for t in range(cfg.iterations)]
    return state, PosteriorEstimate(mu, s, None), diagnostics


def run_cofem_sharded(problem, cfg, device=0, sharded=None):
    """run_cofem (cofem.py:136-157) with the dictionary sharded over the process group.

    Every rank passes the same host problem; each uploads only its shard
    (dense: its columns of Phi; convolution: its samples of y).  Returns the
    full (gathered) PrecisionState, PosteriorEstimate and diagnostics on every
    rank.
    """
    if sharded is None:
        sharded = ShardedContext.for_operator(problem.op, cfg.cg.precision, device)
    c0, c1 = sharded.col_range
    alpha, mu, s, steps, resid = _run_shard(sharded.ctx, problem, cfg, c0, c1)
    return _assemble(cfg, sharded.gather(alpha), sharded.gather(mu), sharded.gather(s), steps, resid)


def run_threaded(world_size, fn, group=None):
    """Run fn(rank) on `world_size` host threads; re-raise the first failure.

    The native calls release the GIL (ctypes), so the ranks' host loops run
    concurrently and meet at the shard group's barriers.  A rank that fails
    aborts `group`, releasing the others."""
    results, errors = [None] * world_size, [None] * world_size

    def body(r):
        try:
            results[r] = fn(r)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errors[r] = e
            if group is not None:
                group.abort()

    threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world_size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for e in errors:
        if e is not None and not isinstance(e, _lib.CofemError):
            raise e
    for e in errors:
        if e is not None:
            raise e
    return results


def threaded_contexts(op, precision, devices):
    """One shard context per entry of `devices`, joined to one in-process
    group (reachable as ``contexts[0].group``)."""
    world = len(devices)
    shards = shard_ranges(op, world)
    group = _lib.ShardGroup(world)
    contexts = []
    for r, (c0, c1) in enumerate(shards):
        ctx = shard_context(op, precision, devices[r], c0, c1)
        ctx.set_group(group, r)
        contexts.append(ctx)
    # the uploads may be collective (float64 ozaki planes): one thread per rank
    run_threaded(world, lambda r: upload_shard(contexts[r], op, *shards[r]), group)
    return contexts, shards


def run_cofem_threaded(problem, cfg, devices=(0, 0)):
    """run_cofem with the dictionary sharded over len(devices) ranks of ONE
    process (one host thread per rank, in-process shard group).  Same results
    layout as run_cofem; the exchanges are those of the NCCL path."""
    contexts, shards = threaded_contexts(problem.op, cfg.cg.precision, list(devices))
    try:
        outs = run_threaded(len(contexts), lambda r: _run_shard(contexts[r], problem, cfg, *shards[r]),
                            contexts[0].group)
    finally:
        for ctx in contexts:
            ctx.close()
    alpha, mu, s = (np.concatenate([o[i] for o in outs]) for i in range(3))
    for o in outs[1:]:  # every rank takes the same PCG decisions
        if not np.array_equal(o[3], outs[0][3]):
            raise RuntimeError("shards disagree on the CG step counts")
    return _assemble(cfg, alpha, mu, s, outs[0][3], outs[0][4])

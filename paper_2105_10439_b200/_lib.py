"""ctypes binding of the C ABI in include/cofem_b200.h.

The shared library is built in-tree (``python -m paper_2105_10439_b200.build``
or ``__graft_entry__.build()``) into ``paper_2105_10439_b200/_lib/``.  There is
no CPU fallback: if the library or a GPU is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int8, c_int32, c_int64, c_uint8, c_uint64, c_void_p

import numpy as np

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib")
LIB_PATH = os.environ.get("COFEM_LIB") or os.path.join(LIB_DIR, "libcofem_b200.so")  # override: profiling variants

COFEM_OK = 0
COFEM_EINVAL = -1
COFEM_ECUDA = -2
COFEM_ENOMEM = -3
COFEM_EDIVERGED = -4
COFEM_ENCCL = -5
COFEM_ESTATE = -6

FP32, FP64, OZAKI, OZAKI24 = 0, 1, 2, 3
THETA_CODES = {"all-ones": 0, "jacobi": 1, "none": 2}
THETA_CUSTOM = 3
VARIANT_CODES = {"standard": 0, "nonneg": 1}

# every symbol include/cofem_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "cofem_abi_version",
    "cofem_last_error",
    "cofem_device_count",
    "cofem_create",
    "cofem_destroy",
    "cofem_create_convolution",
    "cofem_create_dct2",
    "cofem_create_dct1",
    "cofem_set_dictionary",
    "cofem_set_dictionary_f64",
    "cofem_set_shard",
    "cofem_generate_gaussian_dictionary",
    "cofem_get_dictionary",
    "cofem_nccl_get_unique_id",
    "cofem_set_comm",
    "cofem_group_create",
    "cofem_group_destroy",
    "cofem_group_abort",
    "cofem_set_group",
    "cofem_apply",
    "cofem_apply_adjoint",
    "cofem_system_apply",
    "cofem_column_sq_norms",
    "cofem_pcg_solve",
    "cofem_run",
    "cofem_run_multitask",
    "cofem_last_run_report",
    "cofem_pcg_solve_multi",
    "cofem_set_probe_stream",
    "cofem_set_probe_stream_ex",
    "cofem_pcg64_rademacher",
    "cofem_bench_prepare",
    "cofem_bench_iterations",
)


class CgConfigC(ctypes.Structure):
    _fields_ = [("max_steps", c_int32), ("printed_recursion", c_int32), ("tolerance", c_double)]


class CgReportC(ctypes.Structure):
    _fields_ = [
        ("steps_taken", c_int32),
        ("converged", c_int32),
        ("diverged", c_int32),
        ("n_breakdown", c_int32),
        ("final_relative_residual", c_double),
    ]


class EmConfigC(ctypes.Structure):
    _fields_ = [
        ("iterations", c_int32),
        ("probes", c_int32),
        ("variant", c_int32),
        ("theta_policy", c_int32),
        ("clamp_max", c_double),
        ("floor_eps", c_double),
    ]


class TimingC(ctypes.Structure):
    _fields_ = [
        ("total_ms", c_double),
        ("fwd_ms", c_double),
        ("bwd_ms", c_double),
        ("fwd_launches", c_int64),
        ("bwd_launches", c_int64),
        ("pcg_steps", c_int64),
        ("kernel_launches", c_int64),
        ("solve_ms", c_double),
        ("solve_launches", c_int64),
    ]


class CofemError(RuntimeError):
    """A failure reported by the native library (message from cofem_last_error)."""

    def __init__(self, code, msg):
        super().__init__(f"cofem error {code}: {msg}")
        self.code = code


_lib = None


def _dp(a):
    return a.ctypes.data_as(POINTER(c_double))


def load():
    """Load the native library; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2105_10439_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    vp = c_void_p
    sig = {
        "cofem_abi_version": (c_int, []),
        "cofem_last_error": (ctypes.c_char_p, []),
        "cofem_device_count": (c_int, [POINTER(c_int)]),
        "cofem_create": (c_int, [POINTER(vp), c_int, c_int64, c_int64, c_int]),
        "cofem_destroy": (c_int, [vp]),
        "cofem_create_convolution": (c_int, [POINTER(vp), c_int, c_int64, POINTER(c_double), c_int64, c_int]),
        "cofem_create_dct2": (c_int, [POINTER(vp), c_int, c_int64, POINTER(c_int64), c_int64, c_int]),
        "cofem_create_dct1": (c_int, [POINTER(vp), c_int, c_int64, POINTER(c_int64), c_int64, c_int]),
        "cofem_set_dictionary": (c_int, [vp, vp, c_int64, c_int]),
        "cofem_set_dictionary_f64": (c_int, [vp, POINTER(c_double), c_int64]),
        "cofem_set_shard": (c_int, [vp, c_int64, c_int64]),
        "cofem_generate_gaussian_dictionary": (c_int, [vp, c_uint64, c_double]),
        "cofem_get_dictionary": (c_int, [vp, POINTER(c_float)]),
        "cofem_nccl_get_unique_id": (c_int, [vp]),
        "cofem_set_comm": (c_int, [vp, vp, c_int, c_int]),
        "cofem_group_create": (c_int, [POINTER(vp), c_int]),
        "cofem_group_destroy": (c_int, [vp]),
        "cofem_group_abort": (c_int, [vp]),
        "cofem_set_group": (c_int, [vp, vp, c_int]),
        "cofem_apply": (c_int, [vp, POINTER(c_double), c_int64, POINTER(c_double)]),
        "cofem_apply_adjoint": (c_int, [vp, POINTER(c_double), c_int64, POINTER(c_double)]),
        "cofem_system_apply": (c_int, [vp, c_double, POINTER(c_double), POINTER(c_double), c_int64,
                                       POINTER(c_double)]),
        "cofem_column_sq_norms": (c_int, [vp, POINTER(c_double)]),
        "cofem_pcg_solve": (c_int, [vp, c_double, POINTER(c_double), POINTER(c_double), c_int32,
                                    POINTER(c_int32), POINTER(c_double), c_int64, POINTER(CgConfigC),
                                    POINTER(c_double), POINTER(CgReportC), POINTER(c_uint8)]),
        "cofem_run": (c_int, [vp, POINTER(c_double), c_double, POINTER(EmConfigC), POINTER(CgConfigC),
                              POINTER(c_double), POINTER(c_int8), c_uint64, POINTER(c_double),
                              POINTER(c_double), POINTER(c_double), POINTER(c_int32), POINTER(c_double),
                              POINTER(c_int32), POINTER(c_int32)]),
        "cofem_run_multitask": (c_int, [POINTER(vp), c_int, POINTER(POINTER(c_double)), POINTER(c_double),
                                        POINTER(EmConfigC), POINTER(CgConfigC), POINTER(c_double),
                                        POINTER(c_int8), POINTER(c_double), POINTER(POINTER(c_double)),
                                        POINTER(POINTER(c_double)), POINTER(c_int32), POINTER(c_double),
                                        POINTER(c_int32), POINTER(c_int32)]),
        "cofem_last_run_report": (c_int, [vp, c_int32, POINTER(c_double), POINTER(c_double), POINTER(c_uint8),
                                          POINTER(CgReportC)]),
        "cofem_pcg_solve_multi": (c_int, [POINTER(vp), c_int, POINTER(c_double), POINTER(POINTER(c_double)),
                                          POINTER(POINTER(c_double)), POINTER(POINTER(c_double)), POINTER(c_int64),
                                          POINTER(CgConfigC), POINTER(POINTER(c_double)), POINTER(CgReportC),
                                          POINTER(POINTER(c_uint8))]),
        "cofem_set_probe_stream": (c_int, [vp, POINTER(c_uint64), POINTER(c_uint64)]),
        "cofem_set_probe_stream_ex": (c_int, [vp, POINTER(c_uint64), POINTER(c_uint64), c_uint64, c_uint64]),
        "cofem_pcg64_rademacher": (c_int, [c_int, POINTER(c_uint64), POINTER(c_uint64), c_uint64, c_int64, c_int64,
                                           c_int32, POINTER(c_int8)]),
        "cofem_bench_prepare": (c_int, [vp, POINTER(c_double), c_double, POINTER(EmConfigC),
                                        POINTER(CgConfigC), c_uint64]),
        "cofem_bench_iterations": (c_int, [vp, c_int, c_int, POINTER(TimingC)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cofem_abi_version() != 1:
        raise ImportError("libcofem_b200 ABI version mismatch")
    _lib = lib
    return lib


def last_error():
    return load().cofem_last_error().decode(errors="replace")


def check(rc):
    if rc != COFEM_OK:
        raise CofemError(rc, last_error())
    return rc


def device_count():
    n = c_int(0)
    rc = load().cofem_device_count(ctypes.byref(n))
    return n.value if rc == 0 else 0


class Context:
    """Owns one native cofem_ctx: a dense float32 dictionary shard on one GPU."""

    def __init__(self, n_rows, n_cols, precision=FP32, device=0, _handle=None):
        lib = load()
        handle = _handle
        if handle is None:
            handle = c_void_p()
            check(lib.cofem_create(ctypes.byref(handle), int(device), int(n_rows), int(n_cols), int(precision)))
        self._h = handle
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.precision = precision

    @classmethod
    def dct2(cls, n, mask, precision=OZAKI, device=0):
        """Partial 2-D DCT dictionary of n x n images (rows `mask` of the coefficient grid)."""
        mask = np.ascontiguousarray(mask, dtype=np.int64)
        handle = c_void_p()
        check(load().cofem_create_dct2(ctypes.byref(handle), int(device), int(n), mask.ctypes.data_as(POINTER(c_int64)),
                                       mask.size, int(precision)))
        return cls(mask.size, n * n, precision, device, _handle=handle)

    @classmethod
    def dct1(cls, dim, mask, precision=FP64, device=0):
        """1-D subsampled DCT dictionary: rows `mask` of the orthonormal inverse DCT-II of length dim."""
        mask = np.ascontiguousarray(mask, dtype=np.int64)
        handle = c_void_p()
        check(load().cofem_create_dct1(ctypes.byref(handle), int(device), int(dim), mask.ctypes.data_as(POINTER(c_int64)),
                                       mask.size, int(precision)))
        return cls(mask.size, dim, precision, device, _handle=handle)

    @classmethod
    def convolution(cls, dim, taps, precision=OZAKI, device=0):
        """Causal Toeplitz dictionary with the given filter taps (banded int8 path)."""
        taps = np.ascontiguousarray(taps, dtype=np.float64)
        handle = c_void_p()
        check(load().cofem_create_convolution(ctypes.byref(handle), int(device), int(dim), _dp(taps), taps.size,
                                              int(precision)))
        return cls(dim, dim, precision, device, _handle=handle)

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("context already closed")
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None:
            load().cofem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- dictionary
    def set_dictionary_f64(self, phi):
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        if phi.shape != (self.n_rows, self.n_cols):
            raise ValueError(f"dictionary shape {phi.shape} != {(self.n_rows, self.n_cols)}")
        check(load().cofem_set_dictionary_f64(self.handle, _dp(phi), phi.shape[1]))

    def set_dictionary(self, phi):
        phi = np.ascontiguousarray(phi, dtype=np.float32)
        if phi.shape != (self.n_rows, self.n_cols):
            raise ValueError(f"dictionary shape {phi.shape} != {(self.n_rows, self.n_cols)}")
        check(load().cofem_set_dictionary(self.handle, phi.ctypes.data_as(c_void_p), phi.shape[1], 0))

    def set_shard(self, col_offset, global_cols):
        check(load().cofem_set_shard(self.handle, int(col_offset), int(global_cols)))

    def generate_gaussian(self, seed, scale):
        check(load().cofem_generate_gaussian_dictionary(self.handle, int(seed) & (2**64 - 1), float(scale)))

    def get_dictionary(self):
        out = np.empty((self.n_rows, self.n_cols), dtype=np.float32)
        check(load().cofem_get_dictionary(self.handle, out.ctypes.data_as(POINTER(c_float))))
        return out

    def set_comm(self, unique_id: bytes, nranks, rank):
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        check(load().cofem_set_comm(self.handle, ctypes.cast(buf, c_void_p), int(nranks), int(rank)))

    def set_group(self, group, rank):
        """Join an in-process ShardGroup as `rank` (instead of an NCCL communicator)."""
        check(load().cofem_set_group(self.handle, group.handle, int(rank)))
        self.group = group  # the group must outlive its contexts

    # -- operator applications (float64 host blocks)
    def apply(self, V):
        V = np.ascontiguousarray(V, dtype=np.float64)
        if V.ndim != 2 or V.shape[0] != self.n_cols:
            raise ValueError(f"apply: expected ({self.n_cols}, q), got {V.shape}")
        out = np.empty((self.n_rows, V.shape[1]))
        check(load().cofem_apply(self.handle, _dp(V), V.shape[1], _dp(out)))
        return out

    def apply_adjoint(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        if U.ndim != 2 or U.shape[0] != self.n_rows:
            raise ValueError(f"apply_adjoint: expected ({self.n_rows}, q), got {U.shape}")
        out = np.empty((self.n_cols, U.shape[1]))
        check(load().cofem_apply_adjoint(self.handle, _dp(U), U.shape[1], _dp(out)))
        return out

    def system_apply(self, beta, alpha, V):
        V = np.ascontiguousarray(V, dtype=np.float64)
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        out = np.empty_like(V)
        check(load().cofem_system_apply(self.handle, float(beta), _dp(alpha), _dp(V), V.shape[1], _dp(out)))
        return out

    def column_sq_norms(self):
        out = np.empty(self.n_cols)
        check(load().cofem_column_sq_norms(self.handle, _dp(out)))
        return out

    # -- PCG
    def pcg_solve(self, beta, alpha, minv, B, max_steps, tolerance, printed=False, groups=None):
        B = np.ascontiguousarray(B, dtype=np.float64)
        q = B.shape[1]
        alpha = np.ascontiguousarray(alpha, dtype=np.float64)
        minv = np.ascontiguousarray(minv, dtype=np.float64)
        ngroups = 1 if minv.ndim == 1 else minv.shape[1]
        gptr = None
        if ngroups > 1:
            g = np.ascontiguousarray(groups, dtype=np.int32)
            gptr = g.ctypes.data_as(POINTER(c_int32))
        X = np.empty_like(B)
        rep = CgReportC()
        brk = np.zeros(q, dtype=np.uint8)
        cfg = CgConfigC(int(max_steps), 1 if printed else 0, float(tolerance))
        rc = load().cofem_pcg_solve(self.handle, float(beta), _dp(alpha), _dp(minv), ngroups, gptr, _dp(B), q,
                                    ctypes.byref(cfg), _dp(X), ctypes.byref(rep),
                                    brk.ctypes.data_as(POINTER(c_uint8)))
        if rc not in (COFEM_OK, COFEM_EDIVERGED):
            check(rc)
        return X, rep, brk, rc == COFEM_EDIVERGED

    # -- EM loop
    def run(self, y, beta, iterations, probes, variant, theta_policy, clamp_max, floor_eps, max_steps, tolerance,
            printed=False, theta=None, probe_blocks=None, device_probe_seed=0):
        y = np.ascontiguousarray(y, dtype=np.float64)
        em = EmConfigC(int(iterations), int(probes), int(variant), int(theta_policy), float(clamp_max),
                       float(floor_eps))
        cg = CgConfigC(int(max_steps), 1 if printed else 0, float(tolerance))
        th = None
        if theta is not None:
            theta = np.ascontiguousarray(theta, dtype=np.float64)
            th = _dp(theta)
        pr = None
        if probe_blocks is not None:
            probe_blocks = np.ascontiguousarray(probe_blocks, dtype=np.int8)
            assert probe_blocks.shape == (iterations, self.n_cols, probes)
            pr = probe_blocks.ctypes.data_as(POINTER(c_int8))
        d = self.n_cols
        alpha, mu, s = np.empty(d), np.empty(d), np.empty(d)
        steps = np.zeros(iterations, dtype=np.int32)
        resid = np.zeros(iterations)
        fit, fst = c_int32(0), c_int32(0)
        rc = load().cofem_run(self.handle, _dp(y), float(beta), ctypes.byref(em), ctypes.byref(cg), th, pr,
                              int(device_probe_seed) & (2**64 - 1), _dp(alpha), _dp(mu), _dp(s),
                              steps.ctypes.data_as(POINTER(c_int32)), _dp(resid), ctypes.byref(fit),
                              ctypes.byref(fst))
        if rc == COFEM_EDIVERGED:
            return None, (fit.value, fst.value)
        check(rc)
        return (alpha, mu, s, steps, resid), None

    def last_run_report(self, iterations, probes):
        """(wall_times[T], final block X (D x (K+1)), breakdown flags, CgReportC)
        of the last ``run`` (cofem_last_run_report)."""
        wall = np.empty(iterations)
        X = np.empty((self.n_cols, probes + 1))
        brk = np.zeros(probes + 1, dtype=np.uint8)
        rep = CgReportC()
        check(load().cofem_last_run_report(self.handle, int(iterations), _dp(wall), _dp(X),
                                           brk.ctypes.data_as(POINTER(c_uint8)), ctypes.byref(rep)))
        return wall, X, brk, rep

    def set_probe_stream(self, rng, first_half=0, halves_per_iteration=0):
        """Draw the probes on the device from numpy Generator ``rng``'s PCG64
        stream (bit for bit the reference's draw); None restores host probes."""
        if rng is None:
            check(load().cofem_set_probe_stream(self.handle, None, None))
            return
        state, inc = pcg64_words(rng)
        check(load().cofem_set_probe_stream_ex(self.handle, state, inc, int(first_half), int(halves_per_iteration)))

    # -- benchmark hooks
    def bench_prepare(self, y, beta, probes, max_steps, tolerance, theta_policy=0, variant=0, seed=0,
                      clamp_max=1e12, floor_eps=1e-12):
        y = np.ascontiguousarray(y, dtype=np.float64)
        em = EmConfigC(1, int(probes), int(variant), int(theta_policy), float(clamp_max), float(floor_eps))
        cg = CgConfigC(int(max_steps), 0, float(tolerance))
        check(load().cofem_bench_prepare(self.handle, _dp(y), float(beta), ctypes.byref(em), ctypes.byref(cg),
                                         int(seed) & (2**64 - 1)))

    def bench_iterations(self, n_iter, time_kernels=False):
        t = TimingC()
        check(load().cofem_bench_iterations(self.handle, int(n_iter), 1 if time_kernels else 0, ctypes.byref(t)))
        return {k: getattr(t, k) for k, _ in TimingC._fields_}


class ShardGroup:
    """cofem_group: the exchanges of a sharded problem between contexts driven
    from host threads of one process (one thread per rank)."""

    def __init__(self, nranks):
        h = c_void_p()
        check(load().cofem_group_create(ctypes.byref(h), int(nranks)))
        self._h = h
        self.nranks = int(nranks)

    @property
    def handle(self):
        return self._h

    def abort(self):
        """Release ranks waiting at the group's barriers (a rank failed on the host)."""
        check(load().cofem_group_abort(self._h))

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None:
                load().cofem_group_destroy(self._h)
                self._h = None
        except Exception:
            pass


def run_multitask(contexts, ys, betas, iterations, probes, theta_policy, clamp_max, floor_eps, max_steps,
                  tolerance, printed=False, theta=None, probe_blocks=None):
    """cofem_run_multitask over L contexts (one per task, same D, one GPU).

    probe_blocks: T x L x D x K signs or None (every context has a probe
    stream set); theta: L x D (custom policy).  Returns
    ((alpha, mus, ss, steps, resid), None) or (None, (iteration, step)) on divergence."""
    L = len(contexts)
    d = contexts[0].n_cols
    em = EmConfigC(int(iterations), int(probes), 0, int(theta_policy), float(clamp_max), float(floor_eps))
    cg = CgConfigC(int(max_steps), 1 if printed else 0, float(tolerance))
    handles = (c_void_p * L)(*[c.handle for c in contexts])
    ys = [np.ascontiguousarray(y, dtype=np.float64) for y in ys]
    y_ptrs = (POINTER(c_double) * L)(*[_dp(y) for y in ys])
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    assert betas.shape == (L,)
    th = None
    if theta is not None:
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        assert theta.shape == (L, d)
        th = _dp(theta)
    pr = None
    if probe_blocks is not None:
        probe_blocks = np.ascontiguousarray(probe_blocks, dtype=np.int8)
        assert probe_blocks.shape == (iterations, L, d, probes)
        pr = probe_blocks.ctypes.data_as(POINTER(c_int8))
    alpha = np.empty(d)
    mus = [np.empty(d) for _ in range(L)]
    ss = [np.empty(d) for _ in range(L)]
    mu_ptrs = (POINTER(c_double) * L)(*[_dp(m) for m in mus])
    s_ptrs = (POINTER(c_double) * L)(*[_dp(m) for m in ss])
    steps = np.zeros(iterations, dtype=np.int32)
    resid = np.zeros(iterations)
    fit, fst = c_int32(0), c_int32(0)
    rc = load().cofem_run_multitask(handles, L, y_ptrs, _dp(betas), ctypes.byref(em), ctypes.byref(cg), th,
                                    pr, _dp(alpha), mu_ptrs, s_ptrs,
                                    steps.ctypes.data_as(POINTER(c_int32)), _dp(resid), ctypes.byref(fit),
                                    ctypes.byref(fst))
    if rc == COFEM_EDIVERGED:
        return None, (fit.value, fst.value)
    check(rc)
    return (alpha, mus, ss, steps, resid), None


def pcg_solve_multi(contexts, betas, alphas, minvs, Bs, max_steps, tolerance, printed=False):
    """cofem_pcg_solve_multi: block l solves (beta_l Phi_l^T Phi_l + diag(alpha_l)) X_l = B_l
    in one lockstep PCG.  Returns (Xs, CgReportC, breakdown flags per block, diverged)."""
    L = len(contexts)
    handles = (c_void_p * L)(*[c.handle for c in contexts])
    alphas = [np.ascontiguousarray(a, dtype=np.float64) for a in alphas]
    minvs = [np.ascontiguousarray(m, dtype=np.float64) for m in minvs]
    Bs = [np.ascontiguousarray(b, dtype=np.float64) for b in Bs]
    Xs = [np.empty_like(b) for b in Bs]
    brks = [np.zeros(b.shape[1], dtype=np.uint8) for b in Bs]
    betas = np.ascontiguousarray(betas, dtype=np.float64)
    qs = np.array([b.shape[1] for b in Bs], dtype=np.int64)
    ptrs = lambda arrs: (POINTER(c_double) * L)(*[_dp(a) for a in arrs])  # noqa: E731
    bptr = (POINTER(c_uint8) * L)(*[b.ctypes.data_as(POINTER(c_uint8)) for b in brks])
    rep = CgReportC()
    cfg = CgConfigC(int(max_steps), 1 if printed else 0, float(tolerance))
    rc = load().cofem_pcg_solve_multi(handles, L, _dp(betas), ptrs(alphas), ptrs(minvs), ptrs(Bs),
                                      qs.ctypes.data_as(POINTER(c_int64)), ctypes.byref(cfg), ptrs(Xs),
                                      ctypes.byref(rep), bptr)
    if rc not in (COFEM_OK, COFEM_EDIVERGED):
        check(rc)
    return Xs, rep, brks, rc == COFEM_EDIVERGED


def pcg64_words(rng):
    """(state, inc) of a numpy PCG64 Generator as two {hi, lo} uint64 arrays."""
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("the device probe stream reproduces numpy's PCG64 only")
    if st.get("has_uint32"):
        raise ValueError("the generator holds a buffered 32-bit half; draw probes on the host")
    mask = (1 << 64) - 1

    def words(v):
        return (c_uint64 * 2)((v >> 64) & mask, v & mask)

    return words(st["state"]["state"]), words(st["state"]["inc"])


def pcg64_rademacher(rng, half_offset, row0, rows, k, device=0):
    """Rows [row0, row0 + rows) of the D x K sign draw that starts at 32-bit
    half ``half_offset`` of ``rng``'s stream, generated on the GPU (int8)."""
    state, inc = pcg64_words(rng)
    out = np.empty((rows, k), dtype=np.int8)
    check(load().cofem_pcg64_rademacher(int(device), state, inc, int(half_offset), int(row0), int(rows), int(k),
                                        out.ctypes.data_as(POINTER(c_int8))))
    return out


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(load().cofem_nccl_get_unique_id(ctypes.cast(buf, c_void_p)))
    return buf.raw

"""numpy emulation of the Makhoul pair steps of the 2-D DCT passes (csrc/dct.cuh pair_op) in the
lane / slot distribution of the warp-per-FFT passes (csrc/dct1024.cuh): lane lt holds the 32
values lt + 32 r, the pair (k, n - k) meets by a lane exchange, lane 0 through a side buffer.
Test infrastructure (tests/test_host_api.py); nothing in the package imports it."""
import numpy as np
from scipy.fft import dct, idct
N = 1024
lt = np.arange(32)[:, None]; sl = np.arange(32)[None, :]
def fft_warp(r, sign, scale=1.0):
    # r[lane][n2] = x[lane + 32 n2]
    k = np.arange(32)
    F = np.exp(sign * 2j * np.pi * np.outer(k, k) / 32)
    Y = r @ F  # Y[lt][k2]
    Y = Y * np.exp(sign * 2j * np.pi * lt * sl / N) * scale
    s = Y.T.copy()  # s[k2][n1]
    return s @ F  # [lane=k2][k1] = X[k2 + 32 k1]
def partner(a):  # value of lane (32-lt)%32, slot 31-k1
    return a[(32 - np.arange(32)) % 32][:, ::-1]
def load_v(xa, xb):
    n = lt + 32 * sl
    m = np.where(n < N // 2, 2 * n, 2 * N - 1 - 2 * n)
    return xa[m] + 1j * xb[m]
def store_v(v):
    n = lt + 32 * sl
    m = np.where(n < N // 2, 2 * n, 2 * N - 1 - 2 * n)
    xa = np.zeros(N); xb = np.zeros(N)
    xa[m] = v.real; xb[m] = v.imag
    return xa, xb
tw = np.exp(-1j * np.pi * np.arange(N + 1) / (2 * N))
c0, ck = np.sqrt(1 / N), np.sqrt(2 / N)
def pair_loop(s, fn, fix0):
    """generic lanes: owner slots k1<16 compute (out_k, out_nk); lane 0 via the smem fix."""
    out = s.copy()
    y = partner(s)
    kk = (lt + 32 * sl)
    ok, onk = fn(s[:, :16], y[:, :16], kk[:, :16])
    out[:, :16] = ok
    send = np.zeros_like(s); send[:, :16] = onk
    recv = partner(send)  # lane L slot 31-k1 <- lane 32-L slot k1
    out[:, 16:] = recv[:, 16:]
    # lane 0 fix
    S = s[0].copy()
    R = S.copy()
    for j in range(1, 16):
        a, b = fn(S[j], S[32 - j], 32 * j)
        R[j], R[32 - j] = a, b
    R[0], R[16] = fix0(S[0], S[16])
    out[0] = R
    return out
def fwd_item(xa, xb):
    s = fft_warp(load_v(xa, xb), -1)
    def fn(z, y, k):
        T = ck / 2 * tw[k]
        sa = (z.real + y.real) + 1j * (z.imag - y.imag)
        sb = (z.imag + y.imag) + 1j * (y.real - z.real)
        Xa = T.real * sa.real - T.imag * sa.imag; Xb = T.real * sb.real - T.imag * sb.imag
        Xan = -(T.imag * sa.real + T.real * sa.imag); Xbn = -(T.imag * sb.real + T.real * sb.imag)
        return Xa + 1j * Xb, Xan + 1j * Xbn
    def fix0(z0, z16):
        o16, _ = fn(z16, z16, 512)
        return c0 * z0, o16
    out = pair_loop(s, fn, fix0)
    k = (lt + 32 * sl)
    Xa = np.zeros(N); Xb = np.zeros(N); Xa[k] = out.real; Xb[k] = out.imag
    return Xa, Xb
def inv_item(Xa, Xb):
    k = (lt + 32 * sl)
    s = Xa[k] + 1j * Xb[k]
    def fn(z, y, k):
        a_k, b_k, a_n, b_n = z.real, z.imag, y.real, y.imag
        Wk = np.conj(tw[k]) * ((a_k + b_n) + 1j * (b_k - a_n))
        Wn = tw[k] * ((a_k - b_n) + 1j * (a_n + b_k))
        return Wk, Wn
    def fix0(z0, z16):
        w16, _ = fn(z16, z16, 512)
        return np.sqrt(2.0) * z0, w16
    W = pair_loop(s, fn, fix0)
    v = fft_warp(W, +1, 1 / np.sqrt(2 * N))
    return store_v(v)
def fmi_item(xa, xb, mask):
    s = fft_warp(load_v(xa, xb), -1)
    mk = np.concatenate([mask, [0]]).astype(float)
    def fn(z, y, k):
        T = tw[k] / 2
        sa = (z.real + y.real) + 1j * (z.imag - y.imag)
        sb = (z.imag + y.imag) + 1j * (y.real - z.real)
        ua, ub = T * sa, T * sb
        m1, m2 = mk[k], mk[N - k]
        ua = m1 * ua.real + 1j * m2 * ua.imag; ub = m1 * ub.real + 1j * m2 * ub.imag
        Wa, Wb = np.conj(T) * ua, np.conj(T) * ub
        Zk = (Wa.real - Wb.imag) + 1j * (Wa.imag + Wb.real)
        Zn = (Wa.real + Wb.imag) + 1j * (Wb.real - Wa.imag)
        return Zk, Zn
    def fix0(z0, z16):
        return mk[0] * z0 / 2, mk[512] * z16 / 2
    W = pair_loop(s, fn, fix0)
    v = fft_warp(W, +1, 2.0 / N)
    return store_v(v)
def check(seed=0):
    """max abs errors of the three emulated passes against scipy (orthonormal DCT-II / III)."""
    rng = np.random.default_rng(seed)
    xa, xb = rng.standard_normal(N), rng.standard_normal(N)
    out = {}
    Xa, Xb = fwd_item(xa, xb)
    out["fwd"] = max(np.abs(Xa - dct(xa, norm="ortho")).max(), np.abs(Xb - dct(xb, norm="ortho")).max())
    ya, yb = inv_item(xa, xb)
    out["inv"] = max(np.abs(ya - idct(xa, norm="ortho")).max(), np.abs(yb - idct(xb, norm="ortho")).max())
    for name, mask in (("fmi", (rng.random(N) < 0.3).astype(np.uint8)), ("fmi_ones", np.ones(N, np.uint8)),
                       ("fmi_zeros", np.zeros(N, np.uint8))):
        za, zb = fmi_item(xa, xb, mask)
        out[name] = max(np.abs(za - idct(mask * dct(xa, norm="ortho"), norm="ortho")).max(),
                        np.abs(zb - idct(mask * dct(xb, norm="ortho"), norm="ortho")).max())
    return out


if __name__ == "__main__":
    for k, v in check().items():
        print(k, v)

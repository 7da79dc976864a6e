"""numpy model of the planned CUDA DCT kernels (Makhoul DCT via length-N complex FFT,
two real vectors per complex FFT, FFT as 32 x 32 four-step)."""
import numpy as np
from scipy.fft import dct, idct

N = 1024
w32 = np.exp(-2j * np.pi * np.arange(32) / 32)

def fft_4step(z, sign=-1):
    # z length 1024; x[n1 + 32 n2]
    x = z.reshape(32, 32)            # x[n2][n1]
    # step 1: for each n1, DFT over n2
    k2 = np.arange(32)
    F = np.exp(sign * 2j * np.pi * np.outer(np.arange(32), k2) / 32)  # [n2][k2]
    Y = (x.T @ F)                    # Y[n1][k2]
    # twiddle
    Y = Y * np.exp(sign * 2j * np.pi * np.outer(np.arange(32), k2) / N)
    # step 3: for each k2, DFT over n1 -> X[k2 + 32 k1]
    G = np.exp(sign * 2j * np.pi * np.outer(np.arange(32), np.arange(32)) / 32)  # [n1][k1]
    X = (Y.T @ G)                    # X[k2][k1]
    return X.T.reshape(-1)           # index k1*32 + k2 ... we need k = k2 + 32 k1 -> X.T[k1][k2] -> flat k1*32+k2 = k

def reorder(x):
    v = np.empty_like(x)
    v[: N // 2] = x[0::2]
    v[N // 2:] = x[1::2][::-1]
    return v

def unreorder(v):
    x = np.empty_like(v)
    x[0::2] = v[: N // 2]
    x[1::2] = v[N // 2:][::-1]
    return x

k = np.arange(N)
norm = np.where(k == 0, np.sqrt(1.0 / N), np.sqrt(2.0 / N))
tw = np.exp(-1j * np.pi * k / (2 * N))

def dct2_pair(a, b):
    z = reorder(a) + 1j * reorder(b)
    Z = fft_4step(z)
    Zc = np.conj(Z[(-k) % N])
    Va = (Z + Zc) / 2
    Vb = (Z - Zc) / (2j)
    return norm * np.real(tw * Va), norm * np.real(tw * Vb)

def dct3_pair(A, B):
    # inverse of orthonormal DCT-II: W[k] = e^{i pi k/2N} (Xs[k] - i Xs[N-k]), Xs = X / norm ... (Xs[N] = 0)
    def spec(X):
        Xs = X / norm
        Xr = np.zeros(N); Xr[1:] = Xs[::-1][:-1]   # Xs[N-k] for k>=1, 0 for k=0
        return np.conj(tw) * (Xs - 1j * Xr) / N
    W = spec(A) + 1j * spec(B)
    v = fft_4step(W, sign=+1)   # unnormalised inverse DFT
    return unreorder(np.real(v)), unreorder(np.imag(v))

rng = np.random.default_rng(0)
a, b = rng.standard_normal(N), rng.standard_normal(N)
Xa, Xb = dct2_pair(a, b)
print("dct2", np.abs(Xa - dct(a, norm="ortho")).max(), np.abs(Xb - dct(b, norm="ortho")).max())
ya, yb = dct3_pair(Xa, Xb)
print("dct3", np.abs(ya - a).max(), np.abs(yb - b).max())
A, B = rng.standard_normal(N), rng.standard_normal(N)
ya, yb = dct3_pair(A, B)
print("dct3 vs scipy", np.abs(ya - idct(A, norm="ortho")).max(), np.abs(yb - idct(B, norm="ortho")).max())

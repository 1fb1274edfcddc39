"""Seeded synthetic inputs for the BASELINE.json configs; generated on the host
with the reference's generators (SplitMix64 / NormalSampler, rng.hpp:10-39) through the C++ host
library, so the oracle and the device see identical bytes. Not part of any timed region.

There is no public dataset for this path: every config is synthetic, with the shapes, sizes and
value distributions BASELINE.json names.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_HOST = Path(__file__).resolve().parent / "_lib" / "libparfrac_gen.so"  # host only: no CUDA engine
_lib = None


def _host():
    global _lib
    if _lib is None:
        if not _HOST.exists():
            # plain C++ (seconds with g++): rebuild it in-tree rather than fail when a copy of the tree
            # arrives without it; the CUDA engine is never rebuilt implicitly
            from . import build

            try:
                build.build_gen()
            except Exception as e:  # noqa: BLE001
                raise ImportError("libparfrac_gen.so missing and not buildable: %s" % e) from None
        _lib = C.CDLL(str(_HOST))
        _lib.pf_gen_randn.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        _lib.pf_gen_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_void_p]
        _lib.pf_gen_randn_batch.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_void_p, C.c_int]
    return _lib


def randn(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _host().pf_gen_randn(seed, count, out.ctypes.data)
    return out


def uniform(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _host().pf_gen_uniform(seed, count, out.ctypes.data)
    return out


def randn_matrix(n: int, seed: int) -> np.ndarray:
    """make_dense_matrix({Randn, n, seed}) (cli.cpp:40-45): row-major fill."""
    return randn(seed, n * n).reshape(n, n)


def one_norm(m: np.ndarray) -> float:
    """Max column sum, rows accumulated in ascending order (dense.cpp:54-62)."""
    return float(np.max(np.cumsum(np.abs(m), axis=-2)[..., -1, :], axis=-1)) if m.ndim == 2 else None


def one_norms(ms: np.ndarray) -> np.ndarray:
    return np.max(np.cumsum(np.abs(ms), axis=-2)[..., -1, :], axis=-1)


def scaled_to_one_norm(m: np.ndarray, target: float) -> np.ndarray:
    """m.scale(target / m.one_norm()) (test_dense.cpp:19-22)."""
    s = target / one_norm(m)
    return m * s


def cauchy(n: int) -> np.ndarray:
    i = np.arange(n, dtype=np.float64)
    d = i[:, None] - i[None, :]
    return 1.0 / (1.0 + d * d)


def trid121_dense(n: int) -> np.ndarray:
    """TridiagMatrix::trid121(n).to_dense() (action.cpp:27-33, 49-57)."""
    m = np.zeros((n, n))
    idx = np.arange(n)
    m[idx, idx] = 2.0
    m[idx[:-1], idx[:-1] + 1] = -1.0
    m[idx[1:], idx[1:] - 1] = -1.0
    return m


# ------------------------------------------------------------------------------------------ configs


def cfg1() -> np.ndarray:
    """expm of one 64x64, iid N(0,1) from seed 1, rescaled to 1-norm 2.0."""
    return scaled_to_one_norm(randn_matrix(64, 1), 2.0)


def cfg2(batch: int = 4096, n: int = 128, seed0: int = 1000, norm_seed: int = 7, threads: int = 8) -> np.ndarray:
    """batch x n x n, matrix b = NormalSampler(seed0 + b), rescaled to 1-norm 0.5 + 7.5 u_b with
    u_b ~ SplitMix64(norm_seed) (uniform in [0.5, 8])."""
    out = np.empty((batch, n, n), dtype=np.float64)
    _host().pf_gen_randn_batch(seed0, batch, n, out.ctypes.data, threads)
    targets = 0.5 + 7.5 * uniform(norm_seed, batch)
    norms = one_norms(out)
    out *= (targets / norms)[:, None, None]
    return out


def cfg3(n: int = 4096, seed: int = 3, target: float = 16.0) -> np.ndarray:
    """t A with A = -(L + 0.1 R), L = trid121 * n^2 dense, R = N(0,1)/sqrt(n); ||tA||_1 = target."""
    L = trid121_dense(n) * float(n * n)
    R = randn_matrix(n, seed) / np.sqrt(n)
    A = -(L + 0.1 * R)
    return A * (target / one_norm(A))


def cfg4(n: int = 16384, k: int = 64, seed_a: int = 4, seed_v: int = 5, target: float = 4.0):
    """(t A, V): A = N(0,1)/sqrt(n) - 2I, V n x k N(0,1), ||tA||_1 = target."""
    A = randn_matrix(n, seed_a) / np.sqrt(n)
    A[np.arange(n), np.arange(n)] -= 2.0
    A *= target / one_norm(A)
    V = randn(seed_v, n * k).reshape(n, k)
    return A, V


def householder_q(n: int, seed: int) -> np.ndarray:
    """Q of a Householder QR of an n x n seeded Gaussian (numpy/LAPACK geqrf, host, once)."""
    G = randn_matrix(n, seed)
    q, r = np.linalg.qr(G)
    return q * np.sign(np.diag(r))[None, :]


def cfg5(batch: int = 256, n: int = 512, seed_q: int = 11, seed_l: int = 13, lam_max: float = 50.0) -> np.ndarray:
    """batch x n x n symmetric A = Q diag(lambda) Q^T, one shared Q, lambda_b ~ U[0, lam_max]
    from SplitMix64(seed_l) (t = 1)."""
    Q = householder_q(n, seed_q)
    lam = lam_max * uniform(seed_l, batch * n).reshape(batch, n)
    A = np.einsum("ij,bj,kj->bik", Q, lam, Q, optimize=True)
    return 0.5 * (A + np.transpose(A, (0, 2, 1)))

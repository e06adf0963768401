"""TMC oracle — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around oracle/tmc_oracle.cpp, the plain fp64 CPU implementation
of the TMC estimator and its
gradient.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  It shares no code with the
CUDA path (paper_1806_08593_b200/) and never imports it.

Parity status of each routine:
  logsumexp / logmmexp : pinned (closed forms S:56-58, A2 counterexample)
  factor               : pinned (scipy.stats.norm.logpdf, hand-computed D=1 case)
  estimate (value)     : pinned (brute force over all prod K_i combinations, K=1 ELBO,
                          W=0 decoupling, MC unbiasedness vs closed-form p(x))
  estimate (gradients) : pinned (brute-force pair marginals, central finite differences
                          of the brute-force value)
  iwae (NEXT-3)        : pinned (diagonal tuples of the brute-force enumeration, finite
                          differences of that value, K=1 == TMC K=1, E[exp L] = p(x) on C0)
  sample_normal (row a1): pinned (Philox4x32-10 known-answer vectors, ln/cos/sin polynomial
                          accuracy vs numpy, N(0,1) moments and Kolmogorov-Smirnov)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Dict, List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tmc_oracle.cpp")
_LIB = os.path.join(_HERE, "libtmc_oracle.so")
_lib = None

DIR_DOWN = 1
DIR_UP = 2


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               "-fno-fast-math", "-ffp-contract=off", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.or_logsumexp.restype = ctypes.c_double
        _lib.or_logsumexp.argtypes = [P, ctypes.c_int64]
        _lib.or_logmmexp.argtypes = [P, P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, P]
        _lib.or_factor.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int, P, P, P, P, P]
        _lib.or_estimate.argtypes = ([ctypes.c_int, ctypes.c_int, P, P, P] + [P] * 6 +
                                     [ctypes.c_int, P, P] + [P] * 6 + [ctypes.c_int, ctypes.c_double])
        _lib.or_iwae.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P] + [P] * 5 + [P, P] + [P] * 5
        _lib.or_sample_normal.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_int64,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        _lib.or_philox4x32_10.argtypes = [P, P, P]
        _lib.or_log_fp32.restype = ctypes.c_float
        _lib.or_log_fp32.argtypes = [ctypes.c_float]
        _lib.or_cos_sin_2pi.argtypes = [ctypes.c_float, P, P]
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _ptr_array(arrs: List[Optional[np.ndarray]]):
    if arrs is None:
        return None, None
    buf = (ctypes.c_void_p * len(arrs))(*[None if a is None else a.ctypes.data for a in arrs])
    return buf, arrs  # keep arrays alive


def logsumexp(x) -> float:
    x = np.ascontiguousarray(x, np.float64)
    return _load().or_logsumexp(_ptr(x), x.size)


def logmmexp(X, Y) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    I, J = X.shape
    J2, K = Y.shape
    assert J == J2
    Z = np.empty((I, K), np.float64)
    _load().or_logmmexp(_ptr(X), _ptr(Y), I, J, K, _ptr(Z))
    return Z


def _graph(parent, K, D):
    return (np.ascontiguousarray(parent, np.int32), np.ascontiguousarray(K, np.int32),
            np.ascontiguousarray(D, np.int32))


def factor(parent, K, D, i, z, mu, logvar, logq) -> np.ndarray:
    p, k, d = _graph(parent, K, D)
    n = len(p)
    B = z.shape[0]
    Kp = 1 if p[i] < 0 else k[p[i]]
    out = np.empty((B, k[i], Kp), np.float64)
    arrs = [np.ascontiguousarray(a, np.float32) for a in (z, mu, logvar, logq)]
    rc = _load().or_factor(n, B, _ptr(p), _ptr(k), _ptr(d), i, *[_ptr(a) for a in arrs], _ptr(out))
    if rc != 0:
        raise ValueError(f"or_factor failed: {rc}")
    return out


def estimate(parent, K, D, z, mu, logvar, logq, logobs, *, logf_dense=None, direction="up",
             dlogp=None, grads=True, pair=False, threads: Optional[int] = None,
             alpha: float = 1.0) -> Dict[str, object]:
    """Run the oracle.  Inputs are per-latent lists of float32 arrays (tmc_workload layout).

    Returns {"logp": float64[B], and if grads: "dz","dmu","dlogvar","dlogq","dlogobs" lists of
    float64 arrays, and if pair: "pair" list of float64[B][K_i][K_p]}.
    alpha: factor power (every log-factor and observation term times alpha; alpha = 2 gives the
    squared-weight estimate log((1/prod K) sum w^2) of the DReGs surrogate).
    """
    p, k, d = _graph(parent, K, D)
    n = len(p)
    dense = logf_dense is not None
    B = (logf_dense[0] if dense else z[0]).shape[0]
    f32 = lambda lst: None if lst is None else [None if a is None else np.ascontiguousarray(a, np.float32) for a in lst]
    z, mu, logvar, logq, logobs = f32(z), f32(mu), f32(logvar), f32(logq), f32(logobs)
    logf_dense = f32(logf_dense)
    Kp = [1 if p[i] < 0 else int(k[p[i]]) for i in range(n)]
    logp = np.empty(B, np.float64)
    out: Dict[str, object] = {"logp": logp}
    keep = []

    def arr(lst):
        b, a = _ptr_array(lst)
        keep.append(a)
        return b

    gz = gmu = gv = gq = go = pr = None
    if grads:
        go = [np.zeros((B, k[i])) for i in range(n)]
        out["dlogobs"] = go
        if not dense:
            gz = [np.zeros((B, k[i], d[i])) for i in range(n)]
            gmu = [np.zeros((B, Kp[i], d[i])) for i in range(n)]
            gv = [np.zeros((B, Kp[i], d[i])) for i in range(n)]
            gq = [np.zeros((B, k[i])) for i in range(n)]
            out.update(dz=gz, dmu=gmu, dlogvar=gv, dlogq=gq)
    if pair:
        pr = [np.zeros((B, k[i], Kp[i])) for i in range(n)]
        out["pair"] = pr
    dl = None if dlogp is None else np.ascontiguousarray(dlogp, np.float64)
    dirc = {"down": DIR_DOWN, "up": DIR_UP}[direction]
    nt = threads if threads is not None else (os.cpu_count() or 1)
    rc = _load().or_estimate(
        n, B, _ptr(p), _ptr(k), _ptr(d),
        arr(z), arr(mu), arr(logvar), arr(logq), arr(logobs), arr(logf_dense),
        dirc, _ptr(dl), _ptr(logp),
        arr(pr), arr(gz), arr(gmu), arr(gv), arr(gq), arr(go), int(nt), float(alpha))
    if rc != 0:
        raise ValueError(f"or_estimate failed: {rc}")
    return out


def iwae(parent, K, D, z, mu, logvar, logq, logobs, dlogp=None, grads=True) -> Dict[str, object]:
    """IWAE at equal K by its definition, fp64, with gradients."""
    p, k, d = _graph(parent, K, D)
    n = len(p)
    f32 = lambda lst: None if lst is None else [None if a is None else np.ascontiguousarray(a, np.float32) for a in lst]
    z, mu, logvar, logq, logobs = f32(z), f32(mu), f32(logvar), f32(logq), f32(logobs)
    B = z[0].shape[0]
    Kp = [1 if p[i] < 0 else int(k[p[i]]) for i in range(n)]
    out: Dict[str, object] = {"logp": np.empty(B, np.float64)}
    keep = []

    def arr(lst):
        b, a = _ptr_array(lst)
        keep.append(a)
        return b
    gz = gmu = gv = gq = go = None
    if grads:
        gz = [np.zeros((B, k[i], d[i])) for i in range(n)]
        gmu = [np.zeros((B, Kp[i], d[i])) for i in range(n)]
        gv = [np.zeros((B, Kp[i], d[i])) for i in range(n)]
        gq = [np.zeros((B, k[i])) for i in range(n)]
        go = [np.zeros((B, k[i])) for i in range(n)]
        out.update(dz=gz, dmu=gmu, dlogvar=gv, dlogq=gq, dlogobs=go)
    dl = None if dlogp is None else np.ascontiguousarray(dlogp, np.float64)
    rc = _load().or_iwae(n, B, _ptr(p), _ptr(k), _ptr(d), arr(z), arr(mu), arr(logvar), arr(logq), arr(logobs),
                         _ptr(dl), _ptr(out["logp"]), arr(gz), arr(gmu), arr(gv), arr(gq), arr(go))
    if rc != 0:
        raise ValueError(f"or_iwae failed: {rc}")
    return out


def sample_normal(seed: int, tag: int, B: int, b0: int, latent: int, K: int, D: int) -> np.ndarray:
    """Host definition of the reparameterisation noise (include/tmc.h tmc_sample_normal; row a1)."""
    out = np.empty((B, K, D), np.float32)
    if _load().or_sample_normal(int(seed), int(tag), int(B), int(b0), int(latent), int(K), int(D), _ptr(out)) != 0:
        raise ValueError("or_sample_normal failed")
    return out


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    o = np.empty(4, np.uint32)
    _load().or_philox4x32_10(_ptr(c), _ptr(k), _ptr(o))
    return o


def log_fp32(u: float) -> float:
    return float(_load().or_log_fp32(float(u)))


def cos_sin_2pi(v: float):
    c, s = ctypes.c_float(), ctypes.c_float()
    _load().or_cos_sin_2pi(float(v), ctypes.byref(c), ctypes.byref(s))
    return c.value, s.value


def estimate_workload(wl, **kw) -> Dict[str, object]:
    """Convenience: run the oracle on a tmc_workload.Workload."""
    return estimate(wl.parent, wl.K, wl.D, wl.z, wl.mu, wl.logvar, wl.logq, wl.logobs, **kw)

"""paper_1806_08593_b200 — B200-native Tensor Monte Carlo hot path (arXiv 1806.08593).

Thin ctypes binding over libtmc.so (include/tmc.h).  The binding only marshals arguments:
every step of the estimator runs in the library's sm_100a kernels.  torch is used for device
memory and the current CUDA stream only.  There is no CPU fallback: if libtmc.so is missing
or the device is not sm_100a, calls raise.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Dict, List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TMC_LIB_PATH") or os.path.join(_HERE, "libtmc.so")

TMC_DIR_AUTO, TMC_DIR_DOWN, TMC_DIR_UP = 0, 1, 2
TMC_PREC_AUTO, TMC_PREC_SIMT, TMC_PREC_TC = 0, 1, 2
TMC_FLAG_VALIDATE = 1
TMC_FLAG_DENSE_REVERSE = 2
TMC_FLAG_TWO_PASS_REVERSE = 4
TMC_FLAG_SINGLE_PASS_REVERSE = 8

STATUS = {0: "TMC_OK", -1: "TMC_ERR_INVALID_ARG", -2: "TMC_ERR_SHAPE", -3: "TMC_ERR_GRAPH",
          -4: "TMC_ERR_ALIGNMENT", -5: "TMC_ERR_WORKSPACE", -6: "TMC_ERR_UNSUPPORTED_DEVICE",
          -7: "TMC_ERR_CUDA", -8: "TMC_ERR_NONFINITE"}

EXPORTS = ["tmc_workspace_size", "tmc_factors", "tmc_forward", "tmc_backward", "tmc_estimate",
           "tmc_forward_children", "tmc_forward_root", "tmc_sample_normal",
           "tmc_iwae_workspace_size", "tmc_iwae",
           "tmc_estimate_host_workspace_size", "tmc_estimate_host",
           "tmc_last_error", "tmc_version", "tmc_launch_count", "tmc_profile_begin", "tmc_profile_end",
           "tmc_elim_workspace_size", "tmc_elim_forward", "tmc_elim_backward"]


class TmcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class tmc_graph(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("B", ctypes.c_int32),
                ("parent", ctypes.POINTER(ctypes.c_int32)), ("K", ctypes.POINTER(ctypes.c_int32)),
                ("D", ctypes.POINTER(ctypes.c_int32)), ("direction", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("flags", ctypes.c_uint32), ("factor_power", ctypes.c_float)]


class tmc_latent_in(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in ("z", "mu", "logvar", "logq", "logobs")]


class tmc_factor_graph(ctypes.Structure):
    _fields_ = [("nvar", ctypes.c_int32), ("B", ctypes.c_int32), ("K", ctypes.POINTER(ctypes.c_int32)),
                ("nfac", ctypes.c_int32), ("arity", ctypes.POINTER(ctypes.c_int32)),
                ("scope", ctypes.POINTER(ctypes.c_int32)), ("order", ctypes.POINTER(ctypes.c_int32))]


class tmc_profile_entry(ctypes.Structure):
    _fields_ = [("family", ctypes.c_char_p), ("launches", ctypes.c_uint64), ("ms", ctypes.c_double),
                ("mma_flops", ctypes.c_double)]


class tmc_latent_grad(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs", "pair_marginal")]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libtmc.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"libtmc.so not found at {path}; run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        G = ctypes.POINTER(tmc_graph)
        lib.tmc_workspace_size.restype = ctypes.c_size_t
        lib.tmc_workspace_size.argtypes = [G]
        lib.tmc_factors.argtypes = [G, ctypes.c_int32, ctypes.POINTER(tmc_latent_in), P, P]
        lib.tmc_forward.argtypes = [G, ctypes.POINTER(tmc_latent_in), P, P, P, ctypes.c_size_t, P]
        lib.tmc_backward.argtypes = [G, ctypes.POINTER(tmc_latent_in), P, P, ctypes.c_size_t, P,
                                     ctypes.POINTER(tmc_latent_grad), P, P]
        lib.tmc_estimate.argtypes = [G, ctypes.POINTER(tmc_latent_in), P, P,
                                     ctypes.POINTER(tmc_latent_grad), P, ctypes.c_size_t, P]
        lib.tmc_estimate_host_workspace_size.restype = ctypes.c_size_t
        lib.tmc_estimate_host_workspace_size.argtypes = [G, ctypes.c_int32]
        lib.tmc_estimate_host.argtypes = [G, ctypes.POINTER(tmc_latent_in), P, P, ctypes.POINTER(tmc_latent_grad),
                                          ctypes.c_int32, P, ctypes.c_size_t, P]
        lib.tmc_forward_children.argtypes = [G, ctypes.POINTER(tmc_latent_in), P, P, ctypes.c_size_t, P]
        lib.tmc_forward_root.argtypes = [G, ctypes.POINTER(tmc_latent_in), P, P, P, ctypes.c_size_t, P]
        lib.tmc_sample_normal.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_int64,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
        lib.tmc_iwae_workspace_size.restype = ctypes.c_size_t
        lib.tmc_iwae_workspace_size.argtypes = [G]
        lib.tmc_iwae.argtypes = [G, ctypes.POINTER(tmc_latent_in), P, P, ctypes.POINTER(tmc_latent_grad), P,
                                 ctypes.c_size_t, P]
        for f in ("tmc_factors", "tmc_forward", "tmc_backward", "tmc_estimate", "tmc_estimate_host",
                  "tmc_forward_children", "tmc_forward_root", "tmc_sample_normal", "tmc_iwae"):
            getattr(lib, f).restype = ctypes.c_int
        lib.tmc_last_error.restype = ctypes.c_char_p
        lib.tmc_version.restype = ctypes.c_int32
        lib.tmc_launch_count.restype = ctypes.c_uint64
        FG = ctypes.POINTER(tmc_factor_graph)
        lib.tmc_elim_workspace_size.restype = ctypes.c_size_t
        lib.tmc_elim_workspace_size.argtypes = [FG]
        lib.tmc_elim_forward.restype = ctypes.c_int
        lib.tmc_elim_forward.argtypes = [FG, P, P, P, ctypes.c_size_t, P]
        lib.tmc_elim_backward.restype = ctypes.c_int
        lib.tmc_elim_backward.argtypes = [FG, P, P, P, ctypes.c_size_t, P, P, P]
        lib.tmc_profile_begin.restype = ctypes.c_int32
        lib.tmc_profile_begin.argtypes = []
        lib.tmc_profile_end.restype = ctypes.c_int32
        lib.tmc_profile_end.argtypes = [ctypes.POINTER(tmc_profile_entry), ctypes.c_int32]
        _lib = lib
    return _lib


def _check(rc: int):
    if rc != 0:
        raise TmcError(rc, load_library().tmc_last_error().decode())


@dataclasses.dataclass
class Graph:
    """Host-side graph metadata (tmc_graph)."""
    parent: Sequence[int]
    K: Sequence[int]
    D: Sequence[int]
    B: int
    direction: int = TMC_DIR_AUTO
    precision: int = TMC_PREC_AUTO
    flags: int = 0
    factor_power: float = 1.0     # alpha: 2 gives log((1/prod K) sum w^2) (DReGs)

    def __post_init__(self):
        n = len(self.parent)
        self._arrs = [(ctypes.c_int32 * n)(*[int(v) for v in a]) for a in (self.parent, self.K, self.D)]
        self._c = tmc_graph(n, int(self.B), self._arrs[0], self._arrs[1], self._arrs[2],
                            int(self.direction), int(self.precision), int(self.flags), float(self.factor_power))

    @property
    def n(self) -> int:
        return len(self.parent)

    def Kp(self, i: int) -> int:
        return 1 if self.parent[i] < 0 else int(self.K[self.parent[i]])

    def ref(self):
        return ctypes.byref(self._c)


def _dp(t) -> Optional[int]:
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return t.data_ptr()
    return int(t)


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(getattr(stream, "cuda_stream", stream))


def _inputs(inputs: List[Dict]):
    arr = (tmc_latent_in * len(inputs))()
    for j, d in enumerate(inputs):
        for k in ("z", "mu", "logvar", "logq", "logobs"):
            setattr(arr[j], k, _dp(d.get(k)))
    return arr


def _grads(grads: Optional[List[Dict]], n: int):
    arr = (tmc_latent_grad * n)()
    if grads is not None:
        for j, d in enumerate(grads):
            for k in ("dz", "dmu", "dlogvar", "dlogq", "dlogobs", "pair_marginal"):
                setattr(arr[j], k, _dp(d.get(k)) if d else None)
    return arr


def _ptrs(ts):
    if ts is None:
        return None
    return (ctypes.c_void_p * len(ts))(*[_dp(t) for t in ts])


# ----------------------------------------------------------------------------- C-ABI mirrors
def tmc_workspace_size(graph: Graph) -> int:
    n = load_library().tmc_workspace_size(graph.ref())
    if n == 0:
        raise TmcError(-2, load_library().tmc_last_error().decode())
    return n


def tmc_factors(graph: Graph, i: int, inp: Dict, logf, stream=None) -> None:
    one = _inputs([inp])
    _check(load_library().tmc_factors(graph.ref(), int(i), one, _dp(logf), _stream(stream)))


def tmc_forward(graph: Graph, inputs: List[Dict], logp, ws, logf_dense=None, stream=None) -> None:
    _check(load_library().tmc_forward(graph.ref(), _inputs(inputs), _ptrs(logf_dense), _dp(logp),
                                      _dp(ws), ws.numel() * ws.element_size(), _stream(stream)))


def tmc_backward(graph: Graph, inputs: List[Dict], ws, dlogp, grads: Optional[List[Dict]],
                 logf_dense=None, dlogf_dense=None, stream=None) -> None:
    _check(load_library().tmc_backward(graph.ref(), _inputs(inputs), _ptrs(logf_dense), _dp(ws),
                                       ws.numel() * ws.element_size(), _dp(dlogp),
                                       _grads(grads, graph.n), _ptrs(dlogf_dense), _stream(stream)))


def tmc_estimate(graph: Graph, inputs: List[Dict], logp, dlogp, grads: Optional[List[Dict]], ws,
                 stream=None) -> None:
    _check(load_library().tmc_estimate(graph.ref(), _inputs(inputs), _dp(logp), _dp(dlogp),
                                       _grads(grads, graph.n), _dp(ws), ws.numel() * ws.element_size(),
                                       _stream(stream)))


def tmc_forward_children(graph: Graph, inputs: List[Dict], root_msg, ws, stream=None) -> None:
    """Shared-root exchange step 1: root_msg (fp64 [B][K_root+1]) = this shard's child messages."""
    _check(load_library().tmc_forward_children(graph.ref(), _inputs(inputs), _dp(root_msg), _dp(ws),
                                               ws.numel() * ws.element_size(), _stream(stream)))


def tmc_forward_root(graph: Graph, inputs: List[Dict], root_msg_total, logp, ws, stream=None) -> None:
    """Shared-root exchange step 3: the root's elimination from the shard-summed root_msg."""
    _check(load_library().tmc_forward_root(graph.ref(), _inputs(inputs), _dp(root_msg_total), _dp(logp),
                                           _dp(ws), ws.numel() * ws.element_size(), _stream(stream)))


def tmc_iwae(graph: Graph, inputs: List[Dict], logp, dlogp, grads: Optional[List[Dict]], ws, stream=None) -> None:
    """IWAE at equal K on the TMC inputs (NEXT-3): logp [B] fp64 and, if grads, input gradients."""
    _check(load_library().tmc_iwae(graph.ref(), _inputs(inputs), _dp(logp), _dp(dlogp),
                                   None if grads is None else _grads(grads, graph.n), _dp(ws),
                                   ws.numel() * ws.element_size(), _stream(stream)))


def iwae(graph: Graph, inputs: List[Dict], dlogp=None, grads: bool = True, stream=None):
    """Convenience: (logp, grads) of the IWAE estimator; dmu/dlogvar are zero-initialised."""
    import torch
    dev = inputs[0]["z"].device
    logp = torch.empty(graph.B, dtype=torch.float64, device=dev)
    ws = torch.empty(max(1, load_library().tmc_iwae_workspace_size(graph.ref())), dtype=torch.uint8, device=dev)
    g = None
    if grads:
        g = alloc_grads(graph, dev)
        for e in g:
            e["dmu"].zero_()
            e["dlogvar"].zero_()
    tmc_iwae(graph, inputs, logp, dlogp, g, ws, stream)
    return logp, g


# stream tags of the counter-based draws
TAG_PARAMS, TAG_DATA, TAG_PROPOSAL_PARAMS, TAG_EPS, TAG_MC = 1, 2, 3, 4, 5


def tmc_sample_normal(seed: int, tag: int, b0: int, latent: int, eps, stream=None) -> None:
    """eps (device fp32 [B][K][D], contiguous) <- N(0,1) draws of global datapoints b0.. (row a1)."""
    B, K, D = eps.shape
    _check(load_library().tmc_sample_normal(int(seed), int(tag), int(B), int(b0), int(latent), int(K), int(D),
                                            _dp(eps), _stream(stream)))


def tmc_estimate_host_workspace_size(graph: Graph, chunk: int) -> int:
    n = load_library().tmc_estimate_host_workspace_size(graph.ref(), int(chunk))
    if n == 0:
        raise TmcError(-2, load_library().tmc_last_error().decode())
    return n


def tmc_estimate_host(graph: Graph, host_inputs: List[Dict], logp_host, dlogp_host, grads: Optional[List[Dict]],
                      chunk: int, ws, stream=None) -> None:
    """host_inputs / logp_host / dlogp_host: CPU tensors (pinned for overlap); grads: device tensors."""
    _check(load_library().tmc_estimate_host(graph.ref(), _inputs(host_inputs), _dp(logp_host), _dp(dlogp_host),
                                            None if grads is None else _grads(grads, graph.n), int(chunk),
                                            _dp(ws), ws.numel() * ws.element_size(), _stream(stream)))


def tmc_last_error() -> str:
    return load_library().tmc_last_error().decode()


def tmc_version() -> int:
    return load_library().tmc_version()


def tmc_launch_count() -> int:
    return load_library().tmc_launch_count()


@dataclasses.dataclass
class FactorGraph:
    """Host-side metadata of a factor graph over sample indices (tmc_factor_graph, NEXT-4)."""
    K: Sequence[int]
    scopes: Sequence[Sequence[int]]
    B: int
    order: Optional[Sequence[int]] = None

    def __post_init__(self):
        nv, nf = len(self.K), len(self.scopes)
        flat = []
        for sc in self.scopes:
            flat += [int(v) for v in sc] + [0] * (3 - len(sc))
        self._arrs = [(ctypes.c_int32 * nv)(*[int(k) for k in self.K]),
                      (ctypes.c_int32 * nf)(*[len(sc) for sc in self.scopes]),
                      (ctypes.c_int32 * max(1, len(flat)))(*flat)]
        order = None if self.order is None else (ctypes.c_int32 * nv)(*[int(v) for v in self.order])
        self._order = order
        self._c = tmc_factor_graph(nv, int(self.B), self._arrs[0], nf, self._arrs[1], self._arrs[2], order)

    def ref(self):
        return ctypes.byref(self._c)


def tmc_elim_workspace_size(fg: FactorGraph) -> int:
    n = load_library().tmc_elim_workspace_size(fg.ref())
    if n == 0:
        raise TmcError(-2, load_library().tmc_last_error().decode())
    return n


def tmc_elim_forward(fg: FactorGraph, logf, logp, ws, stream=None) -> None:
    """logp (device fp64 [B]) of the factor graph by sequential elimination."""
    _check(load_library().tmc_elim_forward(fg.ref(), _ptrs(logf), _dp(logp), _dp(ws),
                                           ws.numel() * ws.element_size(), _stream(stream)))


def tmc_elim_backward(fg: FactorGraph, logf, logp, ws, dlogp, dlogf, stream=None) -> None:
    """dlogf[j] (device fp32, like logf[j]; None = not wanted) = dJ/dlogf_j (factor marginals)."""
    _check(load_library().tmc_elim_backward(fg.ref(), _ptrs(logf), _dp(logp), _dp(ws),
                                            ws.numel() * ws.element_size(), _dp(dlogp), _ptrs(dlogf),
                                            _stream(stream)))


def eliminate(fg: FactorGraph, logf, dlogp=None, grads: bool = True, stream=None):
    """Convenience: (logp, [dlogf_j]) of a factor graph on the device."""
    import torch
    dev = logf[0].device
    ws = torch.empty(tmc_elim_workspace_size(fg), dtype=torch.uint8, device=dev)
    logp = torch.empty(fg.B, dtype=torch.float64, device=dev)
    tmc_elim_forward(fg, logf, logp, ws, stream)
    dl = None
    if grads:
        dl = [torch.empty_like(f) for f in logf]
        tmc_elim_backward(fg, logf, logp, ws, dlogp, dl, stream)
    return logp, dl


def tmc_profile_begin() -> None:
    """Start recording per-kernel-family device time and issued tensor-core flops (diagnostics)."""
    _check(load_library().tmc_profile_begin())


def tmc_profile_end() -> Dict[str, Dict]:
    """Stop recording; {family: {"launches", "ms", "mma_flops"}} since tmc_profile_begin."""
    arr = (tmc_profile_entry * 16)()
    n = load_library().tmc_profile_end(arr, 16)
    if n < 0:
        _check(n)
    return {arr[i].family.decode(): {"launches": int(arr[i].launches), "ms": float(arr[i].ms),
                                     "mma_flops": float(arr[i].mma_flops)} for i in range(n)}


# ----------------------------------------------------------------------------- convenience
def alloc_workspace(graph: Graph, device="cuda"):
    import torch
    return torch.empty(tmc_workspace_size(graph), dtype=torch.uint8, device=device)


def alloc_grads(graph: Graph, device="cuda", pair: bool = False, dense: bool = False):
    import torch
    out = []
    for i in range(graph.n):
        K, Kp, D = int(graph.K[i]), graph.Kp(i), int(graph.D[i])
        e = dict(dlogobs=torch.empty(graph.B, K, device=device))
        if not dense:
            e.update(dz=torch.empty(graph.B, K, D, device=device),
                     dmu=torch.empty(graph.B, Kp, D, device=device),
                     dlogvar=torch.empty(graph.B, Kp, D, device=device),
                     dlogq=torch.empty(graph.B, K, device=device))
        if pair:
            e["pair_marginal"] = torch.empty(graph.B, K, Kp, device=device)
        out.append(e)
    return out


def estimate(graph: Graph, inputs: List[Dict], dlogp=None, grads: bool = True, pair: bool = False,
             ws=None, stream=None):
    """logp (float64[B]) and, if grads, a list of per-latent gradient dicts (device tensors)."""
    import torch
    dev = inputs[0]["z"].device
    logp = torch.empty(graph.B, dtype=torch.float64, device=dev)
    ws = alloc_workspace(graph, dev) if ws is None else ws
    g = alloc_grads(graph, dev, pair=pair) if grads else None
    if grads:
        tmc_estimate(graph, inputs, logp, dlogp, g, ws, stream)
    else:
        tmc_forward(graph, inputs, logp, ws, None, stream)
    return logp, g

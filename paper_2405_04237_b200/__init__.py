"""paper_2405_04237_b200 -- B200-native distributed FP64 tall-and-skinny QR
(CholeskyQR2, CQR2GS and the modified CQR2GS of arXiv 2405.04237).

Thin ctypes binding of the C ABI in include/tsqr.h (libtsqr.so, built in-tree by
``paper_2405_04237_b200.build``).  The binding only marshals arguments: every step of
the factorisation runs in the library's sm_100a kernels; PyTorch provides device
memory, streams and process groups.  There is no CPU fallback -- importing the
package on a box without the built library raises.

Matrices are FP64 and column-major: use :func:`colmajor_empty` / :func:`to_colmajor`
to build tensors of shape (rows, cols) with strides (1, ld).
"""
from __future__ import annotations

import ctypes
import os
import weakref

from . import build as _build

CQR2, CQR2GS, MCQR2GS, CQR, CQRGS, SCQR3, SCQR, MCQR2GS_ADAPTIVE = 0, 1, 2, 3, 4, 5, 6, 7
ALGOS = {"cqr2": CQR2, "cqr2gs": CQR2GS, "mcqr2gs": MCQR2GS, "cqr": CQR, "cqrgs": CQRGS, "scqr3": SCQR3,
         "scqr": SCQR, "mcqr2gs_adaptive": MCQR2GS_ADAPTIVE}
TSQR_OK, TSQR_ERR_INVALID_ARG, TSQR_ERR_UNSUPPORTED, TSQR_ERR_CUDA = 0, 1, 2, 3
TSQR_ERR_NCCL, TSQR_ERR_BREAKDOWN, TSQR_ERR_WORKSPACE = 4, 5, 6
PLANES = ["local", "nccl", "fused"]
KCLASSES = ["gram", "proj", "update", "trmm", "chol", "small", "allreduce", "cluster"]
PATHS = ["stream", "cluster"]

LIB_PATH = os.environ.get("TSQR_LIB", _build.LIB)  # override: timing experiments only

#: every function declared in include/tsqr.h
EXPORTS = ["tsqr_workspace_bytes", "tsqr_create", "tsqr_factor", "tsqr_wait", "tsqr_last_counts",
           "tsqr_factor_host", "tsqr_set_graph", "tsqr_data_plane", "tsqr_exec_path", "tsqr_set_adapt_tau", "tsqr_skipped_panels", "tsqr_set_lookahead", "tsqr_set_timing", "tsqr_timing_reset", "tsqr_timing", "tsqr_destroy", "tsqr_status_string", "tsqr_last_error", "tsqr_nccl_unique_id",
           "tsqr_nccl_comm_init", "tsqr_nccl_comm_destroy", "tsqr_gram", "tsqr_proj", "tsqr_update",
           "tsqr_chol_inv", "tsqr_trmm"]


class BreakdownInfo(ctypes.Structure):
    _fields_ = [("pass_", ctypes.c_int32), ("panel", ctypes.c_int32), ("stage", ctypes.c_int32),
                ("pivot", ctypes.c_int32), ("pivot_value", ctypes.c_double)]

    def as_dict(self):
        return {"pass": self.pass_, "panel": self.panel, "stage": self.stage, "pivot": self.pivot,
                "pivot_value": self.pivot_value}


class TsqrError(RuntimeError):
    def __init__(self, status: int, msg: str, info: dict | None = None):
        super().__init__(msg)
        self.status = status
        self.info = info


_lib = None
_VP, _I64, _I32, _SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t


def load(build_if_missing: bool = False):
    """Load libtsqr.so (raises if it is absent: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if build_if_missing:
            _build.build()
        else:
            raise ImportError(f"libtsqr.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    L.tsqr_workspace_bytes.argtypes = [_I64, _I32, _I32, _I32, ctypes.c_int]
    L.tsqr_workspace_bytes.restype = _SZ
    L.tsqr_create.argtypes = [ctypes.POINTER(_VP), _I64, _I32, _I32, _VP, ctypes.c_int, _VP, _VP, _SZ]
    L.tsqr_factor.argtypes = [_VP, _VP, _I64, _VP, _I32]
    L.tsqr_wait.argtypes = [_VP, ctypes.POINTER(BreakdownInfo)]
    L.tsqr_last_counts.argtypes = [_VP, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]
    L.tsqr_destroy.argtypes = [_VP]
    L.tsqr_factor_host.argtypes = [_VP, _VP, _I64, _VP, _I32, _VP, _I64, _VP, _I32]
    L.tsqr_set_timing.argtypes = [_VP, _I32]
    L.tsqr_set_graph.argtypes = [_VP, _I32]
    L.tsqr_data_plane.argtypes = [_VP, ctypes.POINTER(_I32)]
    L.tsqr_exec_path.argtypes = [_VP, ctypes.POINTER(_I32)]
    L.tsqr_set_adapt_tau.argtypes = [_VP, ctypes.c_double]
    L.tsqr_set_lookahead.argtypes = [_VP, _I32]
    L.tsqr_skipped_panels.argtypes = [_VP, ctypes.POINTER(_I32)]
    L.tsqr_timing_reset.argtypes = [_VP]
    L.tsqr_timing.argtypes = [_VP, _I32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64),
                              ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    L.tsqr_status_string.argtypes = [ctypes.c_int]
    L.tsqr_status_string.restype = ctypes.c_char_p
    L.tsqr_last_error.restype = ctypes.c_char_p
    L.tsqr_nccl_unique_id.argtypes = [_VP]
    L.tsqr_nccl_comm_init.argtypes = [ctypes.POINTER(_VP), _I32, _I32, _VP, _I32]
    L.tsqr_nccl_comm_destroy.argtypes = [_VP]
    L.tsqr_gram.argtypes = [_VP, _I64, _I64, _I32, _VP, _I32, _VP]
    L.tsqr_proj.argtypes = [_VP, _I64, _VP, _I64, _I64, _I32, _I32, _VP, _I32, _VP]
    L.tsqr_update.argtypes = [_VP, _I64, _VP, _I64, _VP, _I32, _I64, _I32, _I32, _VP]
    L.tsqr_chol_inv.argtypes = [_VP, _I32, _I32, _VP, _I32, _VP, _I32, _VP, _VP]
    L.tsqr_trmm.argtypes = [_VP, _I64, _I64, _I32, _VP, _I32, _VP]
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype or ctypes.c_int
    _lib = L
    return L


def _check(rc: int, what: str, info: dict | None = None):
    if rc != TSQR_OK:
        L = load()
        raise TsqrError(rc, f"{what}: {L.tsqr_status_string(rc).decode()} -- {L.tsqr_last_error().decode()}", info)


# ----------------------------------------------------------------------------- tensors
def colmajor_empty(rows: int, cols: int, ld: int | None = None, device="cuda", dtype=None):
    """Uninitialised (rows x cols) FP64 tensor with strides (1, ld)."""
    import torch
    ld = max(1, rows) if ld is None else ld
    t = torch.empty((cols, ld), dtype=dtype or torch.float64, device=device)
    return t.T[:rows]


def to_colmajor(x, device="cuda", ld: int | None = None):
    """Column-major FP64 copy of a (rows x cols) tensor or numpy array on `device`."""
    import numpy as np
    import torch
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.asarray(x, dtype=np.float64))
    out = colmajor_empty(x.shape[0], x.shape[1], ld=ld, device=device)
    out.copy_(x)
    return out


def _ld(t) -> int:
    import torch
    if t.dtype != torch.float64:
        raise TypeError("FP64 tensors only")
    if t.dim() != 2 or (t.shape[0] > 1 and t.stride(0) != 1):
        raise ValueError("expected a column-major (rows x cols) tensor with stride(0) == 1")
    return max(t.stride(1), 1) if t.shape[1] > 1 else max(t.shape[0], 1)


def _stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


# ----------------------------------------------------------------------------- NCCL
class NcclComm:
    """An NCCL communicator created through the library (tsqr_nccl_comm_init). The 128-byte
    unique id is broadcast with torch.distributed over the default process group."""

    def __init__(self, rank: int, world: int, device: int):
        import torch
        import torch.distributed as dist
        L = load()
        idbuf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _check(L.tsqr_nccl_unique_id(ctypes.cast(idbuf, _VP)), "tsqr_nccl_unique_id")
        t = torch.tensor(list(bytes(idbuf)), dtype=torch.uint8)
        if dist.get_backend() == "nccl":
            t = t.cuda(device)
        dist.broadcast(t, 0)
        raw = bytes(t.cpu().tolist())
        idbuf = (ctypes.c_uint8 * 128).from_buffer_copy(raw)
        comm = _VP()
        _check(L.tsqr_nccl_comm_init(ctypes.byref(comm), world, rank, ctypes.cast(idbuf, _VP), device),
               "tsqr_nccl_comm_init")
        self.handle = comm.value
        self.rank, self.world = rank, world
        self._plans = weakref.WeakSet()  # plans created on this communicator

    def close(self):
        """Destroys the plans still open on this communicator first (a plan's window and device
        communicator must be released while the communicator is alive), then the communicator."""
        if self.handle:
            for p in list(self._plans):
                p.close()
            load().tsqr_nccl_comm_destroy(self.handle)
            self.handle = None


# ----------------------------------------------------------------------------- plans
class Plan:
    """A factorisation plan (tsqr_create); owns the workspace tensor it allocates."""

    def __init__(self, m_local: int, n: int, b: int, algo="mcqr2gs", comm: NcclComm | None = None,
                 stream=None, device=None):
        import torch
        L = load()
        self.algo = ALGOS[algo] if isinstance(algo, str) else int(algo)
        self.m, self.n, self.b = int(m_local), int(n), int(b)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        nranks = comm.world if comm else 1
        nbytes = L.tsqr_workspace_bytes(self.m, self.n, self.b, nranks, self.algo)
        if nbytes == 0:
            _check(TSQR_ERR_INVALID_ARG if self.n > 0 else TSQR_ERR_INVALID_ARG, "tsqr_workspace_bytes")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
        base = self.workspace.data_ptr()
        aligned = (base + 255) // 256 * 256
        h = _VP()
        rc = L.tsqr_create(ctypes.byref(h), self.m, self.n, self.b, comm.handle if comm else None, self.algo,
                           _stream_ptr(self.stream), aligned, nbytes)
        _check(rc, "tsqr_create")
        self.handle = h.value
        if comm is not None:
            comm._plans.add(self)

    def factor(self, A, R=None, wait: bool = True):
        """A (m_local x n, column-major CUDA FP64) is overwritten by Q; returns R (n x n)."""
        L = load()
        if R is None:
            R = colmajor_empty(self.n, self.n, device=self.device)
        if tuple(A.shape) != (self.m, self.n):
            raise ValueError(f"A has shape {tuple(A.shape)}, plan expects {(self.m, self.n)}")
        _check(L.tsqr_factor(self.handle, A.data_ptr(), _ld(A), R.data_ptr(), _ld(R)), "tsqr_factor")
        if wait:
            self.wait()
        return R

    def wait(self):
        L = load()
        info = BreakdownInfo()
        rc = L.tsqr_wait(self.handle, ctypes.byref(info))
        _check(rc, "tsqr_wait", info.as_dict() if rc == TSQR_ERR_BREAKDOWN else None)

    def factor_host(self, A_host, R_host, A_dev, R_dev):
        """End-to-end form: pinned host A (overwritten by Q) -> device -> factor -> host Q, R."""
        L = load()
        _check(L.tsqr_factor_host(self.handle, A_host.data_ptr(), _ld(A_host), R_host.data_ptr(), _ld(R_host),
                                  A_dev.data_ptr(), _ld(A_dev), R_dev.data_ptr(), _ld(R_dev)), "tsqr_factor_host")

    def set_graph(self, on: bool = True):
        _check(load().tsqr_set_graph(self.handle, 1 if on else 0), "tsqr_set_graph")

    def data_plane(self) -> str:
        """'local' (one rank), 'nccl' (k_reduce + ncclAllReduce) or 'fused' (k_reduce_allreduce)."""
        v = _I32()
        _check(load().tsqr_data_plane(self.handle, ctypes.byref(v)), "tsqr_data_plane")
        return PLANES[v.value]

    def exec_path(self) -> str:
        """'stream' (one kernel per step, CUDA graph) or 'cluster' (one-launch small-problem kernel)."""
        v = _I32()
        _check(load().tsqr_exec_path(self.handle, ctypes.byref(v)), "tsqr_exec_path")
        return PATHS[v.value]

    def set_lookahead(self, on: bool = True):
        """NEXT-f1: run each panel's CholeskyQR chain on a second stream under the trailing update."""
        _check(load().tsqr_set_lookahead(self.handle, 1 if on else 0), "tsqr_set_lookahead")

    def set_adapt_tau(self, tau: float):
        """mcqr2gs_adaptive: skip threshold of the repetition rule (0 never skips)."""
        _check(load().tsqr_set_adapt_tau(self.handle, float(tau)), "tsqr_set_adapt_tau")

    def skipped_panels(self) -> int:
        """Panels whose CholeskyQR repetition the last factorisation skipped (after wait)."""
        v = _I32()
        _check(load().tsqr_skipped_panels(self.handle, ctypes.byref(v)), "tsqr_skipped_panels")
        return v.value

    def set_timing(self, on: bool = True):
        _check(load().tsqr_set_timing(self.handle, 1 if on else 0), "tsqr_set_timing")

    def timing_reset(self):
        _check(load().tsqr_timing_reset(self.handle), "tsqr_timing_reset")

    def timing(self) -> dict:
        """Per kernel class: {"ms", "launches", "flops", "bytes"} summed since timing_reset."""
        L = load()
        out = {}
        for c, name in enumerate(KCLASSES):
            ms, n, fl, by = ctypes.c_double(), _I64(), ctypes.c_double(), ctypes.c_double()
            _check(L.tsqr_timing(self.handle, c, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl),
                                 ctypes.byref(by)), "tsqr_timing")
            out[name] = {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}
        return out

    def counts(self) -> tuple[int, int]:
        L = load()
        a, k = _I64(), _I64()
        _check(L.tsqr_last_counts(self.handle, ctypes.byref(a), ctypes.byref(k)), "tsqr_last_counts")
        return a.value, k.value

    def close(self):
        if getattr(self, "handle", None):
            load().tsqr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def factor(A, b: int, algo="mcqr2gs", comm: NcclComm | None = None):
    """One-shot A = QR: A (column-major CUDA FP64, m_local x n) is overwritten by Q; returns R."""
    p = Plan(A.shape[0], A.shape[1], b, algo, comm=comm, device=A.device)
    try:
        return p.factor(A)
    finally:
        p.close()


# ----------------------------------------------------------------------------- step entry points
def gram(X, W=None):
    L = load()
    m, b = X.shape
    W = colmajor_empty(b, b, device=X.device) if W is None else W
    _check(L.tsqr_gram(X.data_ptr(), _ld(X), m, b, W.data_ptr(), _ld(W), _stream_ptr()), "tsqr_gram")
    return W


def proj(Lm, Rm, out=None):
    L = load()
    m, p = Lm.shape
    q = Rm.shape[1]
    out = colmajor_empty(p, q, device=Lm.device) if out is None else out
    _check(L.tsqr_proj(Lm.data_ptr(), _ld(Lm), Rm.data_ptr(), _ld(Rm), m, p, q, out.data_ptr(), _ld(out),
                       _stream_ptr()), "tsqr_proj")
    return out


def update(X, Lm, S):
    L = load()
    m, q = X.shape
    p = Lm.shape[1]
    _check(L.tsqr_update(X.data_ptr(), _ld(X), Lm.data_ptr(), _ld(Lm), S.data_ptr(), _ld(S), m, p, q,
                         _stream_ptr()), "tsqr_update")
    return X


def chol_inv(W):
    """Returns (U, Z=U^{-1}, status[8] int32 tensor)."""
    import torch
    L = load()
    b = W.shape[0]
    U = colmajor_empty(b, b, device=W.device)
    Z = colmajor_empty(b, b, device=W.device)
    st = torch.zeros(8, dtype=torch.int32, device=W.device)
    _check(L.tsqr_chol_inv(W.data_ptr(), _ld(W), b, U.data_ptr(), _ld(U), Z.data_ptr(), _ld(Z), st.data_ptr(),
                           _stream_ptr()), "tsqr_chol_inv")
    return U, Z, st


def trmm(X, Z):
    L = load()
    m, b = X.shape
    _check(L.tsqr_trmm(X.data_ptr(), _ld(X), m, b, Z.data_ptr(), _ld(Z), _stream_ptr()), "tsqr_trmm")
    return X

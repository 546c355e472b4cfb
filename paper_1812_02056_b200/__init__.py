"""stepfact on B200 — thin Python binding over libstepfact.so (include/stepfact.h).

Argument marshalling only: every step of the factorizations runs in the library's CUDA
kernels (sm_100a).  PyTorch supplies device memory and streams.  There is no CPU
fallback: if the shared library is missing or fails to load, importing the binding's
compute functions raises.

Layout: the C ABI is column-major.  A torch tensor T (row-major, contiguous) read as a
column-major buffer is T^T, so:
  * `*_colmajor` functions take buffers that already hold column-major matrices
    (what bench.py uses; no torch kernel runs);
  * `chol(A)`, `lu(A)`, `qr(A)` take ordinary (row-major) torch matrices and return
    ordinary torch matrices, doing the layout transposes with torch (marshalling).
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libstepfact.so")

SF_F64, SF_F32 = 0, 1
_STATUS = {0: "SF_OK", 1: "SF_EINVAL", 2: "SF_ENOTSUP", 3: "SF_ENOMEM", 4: "SF_ECUDA", 5: "SF_ENCCL"}
_lib = None


class StepfactError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


def lib():
    """Load libstepfact.so (built by paper_1812_02056_b200/build.py or __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_1812_02056_b200.build` "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, p, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_double
    sig = {
        "chol_factor": [i64, i64, i32, p, i64, p, i64, p, p],
        "lu_factor": [i64, i64, i32, p, i64, p, i64, p, p],
        "qr_factor": [i64, i64, i32, p, i64, p, i64, p, i64, p, p],
        "chol_factor_host": [i64, i64, i32, p, i64, p, i64, p],
        "lu_factor_host": [i64, i64, i32, p, i64, p, i64, p],
        "qr_factor_host": [i64, i64, i32, p, i64, p, i64, p, i64, p],
        "sf_chol_panel": [i64, i64, i32, p, i64, i64, p, p],
        "sf_syrk_sub": [i64, i64, i32, p, i64, p, i64, p],
        "sf_gemm_sub": [i64, i64, i64, i32, p, i64, i32, p, i64, i32, p, i64, p],
        "sf_lu_panel": [i64, i64, i64, i32, p, i64, i64, dbl, p, p],
        "sf_qr_panel": [i64, i64, i32, p, i64, i64, dbl, p, p],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = i32
    for name, args in {"chol_solve": [i64, i64, i32, p, i64, p, i64, p],
                       "lu_solve": [i64, i64, i32, p, i64, p, i64, p],
                       "qr_solve": [i64, i64, i32, p, i64, p, i64, p, i64, p]}.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = i32
    pi = ctypes.POINTER(ctypes.c_int64)
    for name, args in {"chol_factor_steps": [i64, i64, pi, i32, p, i64, p, i64, p, p],
                       "lu_factor_steps": [i64, i64, pi, i32, p, i64, p, i64, p, p],
                       "qr_factor_steps": [i64, i64, pi, i32, p, i64, p, i64, p, i64, p, p]}.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = i32
    pp = ctypes.POINTER(ctypes.c_void_p)
    dist_sig = {
        "chol_factor_dist": [p, i64, i64, i32, pp, pp, i64, pp, p],
        "lu_factor_dist": [p, i64, i64, i32, pp, pp, i64, pp, p],
        "qr_factor_dist": [p, i64, i64, i32, pp, pp, pp, i64, pp, p],
        "sf_get_unique_id": [p],
        "sf_comm_init": [p, i32, i32, p],
        "sf_comm_init_loopback": [p, i32],
        "sf_comm_destroy": [p],
        "sf_comm_size": [p],
        "sf_comm_local_ranks": [p],
        "sf_comm_set_push": [p, i32],
    }
    for name, args in dist_sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = i32
    L.sf_comm_bcast_bytes.argtypes = [p]
    L.sf_comm_bcast_bytes.restype = i64
    L.sf_local_cols.argtypes = [i64, i64, i32, i32]
    L.sf_local_cols.restype = i64
    L.sf_flush_count.argtypes = [i64, i64]
    L.sf_flush_count.restype = i64
    L.sf_schedule.argtypes = [i64, i64, ctypes.POINTER(ctypes.c_int64), p, i64]
    L.sf_schedule.restype = i64
    L.sf_launch_counter.argtypes = []
    L.sf_launch_counter.restype = i64
    L.sf_set_strassen.argtypes = [i32, i64]
    L.sf_set_strassen.restype = i32
    L.sf_strerror.argtypes = [i32]
    L.sf_strerror.restype = ctypes.c_char_p
    L.sf_last_error.argtypes = []
    L.sf_last_error.restype = ctypes.c_char_p
    L.sf_version.restype = i32
    L.sf_profile_enable.argtypes = [i32]
    L.sf_profile_enable.restype = None
    L.sf_profile_collect.argtypes = [p, p, p]
    L.sf_profile_collect.restype = i32
    L.sf_profile_union.argtypes = [p]
    L.sf_profile_union.restype = i32
    _lib = L
    return L


EXPORTS = ("chol_factor", "lu_factor", "qr_factor", "chol_factor_host", "lu_factor_host", "qr_factor_host",
           "sf_chol_panel", "sf_syrk_sub", "sf_gemm_sub", "sf_lu_panel", "sf_qr_panel", "sf_flush_count",
           "sf_launch_counter", "sf_strerror", "sf_last_error", "sf_version", "sf_profile_enable",
           "sf_profile_collect", "sf_get_unique_id", "sf_comm_init", "sf_comm_init_loopback", "sf_comm_destroy",
           "sf_comm_size", "sf_comm_local_ranks", "sf_local_cols", "chol_factor_dist", "lu_factor_dist",
           "qr_factor_dist", "chol_factor_steps", "lu_factor_steps", "qr_factor_steps", "chol_solve", "lu_solve",
           "qr_solve", "sf_set_strassen", "sf_schedule", "sf_comm_bcast_bytes", "sf_comm_set_push",
           "sf_profile_union")


def _check(rc):
    if rc != 0:
        raise StepfactError(rc, lib().sf_last_error().decode())


def _dtype_code(t):
    import torch
    if t.dtype == torch.float64:
        return SF_F64
    if t.dtype == torch.float32:
        return SF_F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise ValueError("device entry points need CUDA tensors")


def flush_count(n, s):
    return int(lib().sf_flush_count(n, s))


def schedule(n, s):
    """0-based columns at which the library's drivers flush (sf_schedule): s an int (fixed
    step) or a step sequence."""
    seq = [int(s)] if not isinstance(s, (list, tuple)) else [int(x) for x in s]
    arr = (ctypes.c_int64 * len(seq))(*seq)
    cnt = lib().sf_schedule(n, len(seq), arr, None, 0)
    if cnt < 0:
        raise StepfactError(1, "bad schedule arguments")
    out = (ctypes.c_int64 * max(cnt, 1))()
    lib().sf_schedule(n, len(seq), arr, ctypes.addressof(out), cnt)
    return [int(out[i]) for i in range(cnt)]


def launch_counter():
    return int(lib().sf_launch_counter())


def set_strassen(levels, min_dim=4096):
    """sf_set_strassen: Strassen-Winograd (levels 1-3, 0 = off) in fp64 flushes with sides >= min_dim (f1)."""
    _check(lib().sf_set_strassen(int(levels), int(min_dim)))


def profile_enable(on=True):
    lib().sf_profile_enable(1 if on else 0)


def profile_collect():
    """{kind: (ms, count, flops)} for kinds 'update', 'panel', 'qr_r', 'bcast' (flops = bytes)
    since the last collect."""
    ms = (ctypes.c_double * 4)(); cnt = (ctypes.c_int64 * 4)(); fl = (ctypes.c_double * 4)()
    _check(lib().sf_profile_collect(ctypes.addressof(ms), ctypes.addressof(cnt), ctypes.addressof(fl)))
    return {k: (ms[i], cnt[i], fl[i]) for i, k in enumerate(("update", "panel", "qr_r", "bcast"))}


def profile_union():
    """{kind: wall-clock ms of the union of that kind's regions} from the last profile_collect."""
    ms = (ctypes.c_double * 4)()
    _check(lib().sf_profile_union(ctypes.addressof(ms)))
    return {k: ms[i] for i, k in enumerate(("update", "panel", "qr_r", "bcast"))}


# ----------------------------------------------------------------------- raw column-major API

def _ptr(x):
    return x.data_ptr() if hasattr(x, "data_ptr") else int(x)


def _dt(dtype, *bufs):
    """The SF_* dtype code: inferred from the (torch) buffers when not given; every tensor
    buffer must then agree with it (a mismatch would make the library read and write past
    a buffer of the other element size)."""
    import torch
    codes = {torch.float64: SF_F64, torch.float32: SF_F32}
    seen = {codes.get(b.dtype, -1) for b in bufs if hasattr(b, "dtype")}
    if dtype is None:
        if len(seen) != 1 or -1 in seen:
            raise TypeError("buffers must all be float64 or all float32 tensors (or pass dtype=)")
        return seen.pop()
    if seen - {dtype}:
        raise TypeError(f"dtype={dtype} does not match the buffers' element type")
    return dtype


def chol_colmajor(n, s, dA, lda, dL, ldl, d_info, dtype=None, stream=None):
    """chol_factor on raw column-major device buffers (torch tensors or int pointers; with raw
    pointers pass dtype)."""
    dt = _dt(dtype, dA, dL)
    _check(lib().chol_factor(n, s, dt, _ptr(dA), lda, _ptr(dL), ldl, _ptr(d_info), _stream(stream)))


def lu_colmajor(n, s, dA, lda, dLU, ldlu, d_info, dtype=None, stream=None):
    _check(lib().lu_factor(n, s, _dt(dtype, dA, dLU), _ptr(dA), lda, _ptr(dLU), ldlu, _ptr(d_info), _stream(stream)))


def qr_colmajor(n, s, dA, lda, dQ, ldq, dR, ldr, d_info, dtype=None, stream=None):
    _check(lib().qr_factor(n, s, _dt(dtype, dA, dQ, dR), _ptr(dA), lda, _ptr(dQ), ldq, _ptr(dR), ldr, _ptr(d_info),
                           _stream(stream)))


def _steps_arr(steps):
    return (ctypes.c_int64 * len(steps))(*[int(x) for x in steps])


def chol_steps_colmajor(n, steps, dA, lda, dL, ldl, d_info, dtype=None, stream=None):
    """chol_factor_steps: variable step sequence."""
    _check(lib().chol_factor_steps(n, len(steps), _steps_arr(steps), _dt(dtype, dA, dL), _ptr(dA), lda, _ptr(dL), ldl,
                                   _ptr(d_info), _stream(stream)))


def lu_steps_colmajor(n, steps, dA, lda, dLU, ldlu, d_info, dtype=None, stream=None):
    _check(lib().lu_factor_steps(n, len(steps), _steps_arr(steps), _dt(dtype, dA, dLU), _ptr(dA), lda, _ptr(dLU), ldlu,
                                 _ptr(d_info), _stream(stream)))


def qr_steps_colmajor(n, steps, dA, lda, dQ, ldq, dR, ldr, d_info, dtype=None, stream=None):
    _check(lib().qr_factor_steps(n, len(steps), _steps_arr(steps), _dt(dtype, dA, dQ, dR), _ptr(dA), lda, _ptr(dQ), ldq,
                                 _ptr(dR), ldr, _ptr(d_info), _stream(stream)))


def chol_solve_colmajor(n, nrhs, dL, ldl, dB, ldb, dtype=None, stream=None):
    """chol_solve: B := A^-1 B with A = L L^T (column-major device buffers)."""
    _check(lib().chol_solve(n, nrhs, _dt(dtype, dL, dB), _ptr(dL), ldl, _ptr(dB), ldb, _stream(stream)))


def lu_solve_colmajor(n, nrhs, dLU, ldlu, dB, ldb, dtype=None, stream=None):
    _check(lib().lu_solve(n, nrhs, _dt(dtype, dLU, dB), _ptr(dLU), ldlu, _ptr(dB), ldb, _stream(stream)))


def qr_solve_colmajor(n, nrhs, dQ, ldq, dR, ldr, dB, ldb, dtype=None, stream=None):
    _check(lib().qr_solve(n, nrhs, _dt(dtype, dQ, dR, dB), _ptr(dQ), ldq, _ptr(dR), ldr, _ptr(dB), ldb,
                          _stream(stream)))


# ----------------------------------------------------------------------- torch convenience API

def _colmajor_copy(A):
    """Column-major copy of the logical matrix A: buffer B with B.T == A (a torch transpose)."""
    return A.mT.contiguous()


def chol(A, s, stream=None):
    """Cholesky of a symmetric positive definite CUDA matrix A (Alg. 1). Returns (L, info)."""
    import torch
    _need_cuda(A)
    n = A.shape[0]
    B = _colmajor_copy(A)
    L = torch.zeros_like(B)
    info = torch.zeros(1, dtype=torch.int64, device=A.device)
    chol_colmajor(n, s, B, n, L, n, info, _dtype_code(A), stream)
    return L.mT, int(info.item())


def lu(A, s, stream=None):
    """Crout LU without pivoting (Alg. 2). Returns (L, U, info) with U unit upper."""
    import torch
    _need_cuda(A)
    n = A.shape[0]
    B = _colmajor_copy(A)
    info = torch.zeros(1, dtype=torch.int64, device=A.device)
    lu_colmajor(n, s, B, n, B, n, info, _dtype_code(A), stream)
    F = B.mT
    L = torch.tril(F)
    U = torch.triu(F, 1) + torch.eye(n, dtype=A.dtype, device=A.device)
    return L, U, int(info.item())


def qr(A, s, stream=None):
    """QR by Alg. 3 (MGS panels, block projection flushes). Returns (Q, R, info)."""
    import torch
    _need_cuda(A)
    n = A.shape[0]
    B = _colmajor_copy(A)
    Q = torch.empty_like(B)
    R = torch.empty_like(B)
    info = torch.zeros(1, dtype=torch.int64, device=A.device)
    qr_colmajor(n, s, B, n, Q, n, R, n, info, _dtype_code(A), stream)
    return Q.mT, R.mT, int(info.item())


# ----------------------------------------------------------------------- host (end-to-end) API

def _host_buf(x, n, dtype=None):
    """(pointer, SF_* dtype) of an n x n column-major HOST buffer, validated: a numpy array in
    Fortran order (logical matrix X, X[i, j] at column-major offset i + j*n) or a contiguous
    CPU torch tensor holding the column-major buffer (row j = column j, i.e. the tensor is
    X^T).  The element type must be float64 or float32 and agree with `dtype` if given."""
    if hasattr(x, "data_ptr"):
        import torch
        if x.is_cuda or not x.is_contiguous() or tuple(x.shape) != (n, n):
            raise ValueError("host buffers must be contiguous CPU tensors of shape (n, n)")
        code = {torch.float64: SF_F64, torch.float32: SF_F32}.get(x.dtype)
        ptr = x.data_ptr()
    else:
        if not isinstance(x, np.ndarray) or x.shape != (n, n) or not x.flags["F_CONTIGUOUS"]:
            raise ValueError("host buffers must be Fortran-ordered (column-major) numpy arrays of shape (n, n)")
        if not x.flags["WRITEABLE"]:
            raise ValueError("host buffers must be writeable")
        code = {np.dtype(np.float64): SF_F64, np.dtype(np.float32): SF_F32}.get(x.dtype)
        ptr = x.ctypes.data
    if code is None:
        raise TypeError("host buffers must be float64 or float32")
    if dtype is not None and dtype != code:
        raise TypeError(f"dtype={dtype} does not match the host buffer's element type")
    return ptr, code


def chol_host(hA, s, hL=None, dtype=None):
    """chol_factor_host on column-major host buffers (pinned torch tensors or numpy); dtype is
    inferred from hA and every buffer must match it."""
    n = hA.shape[0]
    pa, dt = _host_buf(hA, n, dtype)
    out = hA if hL is None else hL
    po, _ = _host_buf(out, n, dt)
    info = ctypes.c_int64(0)
    _check(lib().chol_factor_host(n, s, dt, pa, n, po, n, ctypes.addressof(info)))
    return out, info.value


def lu_host(hA, s, hLU=None, dtype=None):
    n = hA.shape[0]
    pa, dt = _host_buf(hA, n, dtype)
    out = hA if hLU is None else hLU
    po, _ = _host_buf(out, n, dt)
    info = ctypes.c_int64(0)
    _check(lib().lu_factor_host(n, s, dt, pa, n, po, n, ctypes.addressof(info)))
    return out, info.value


def qr_host(hA, s, hQ, hR, dtype=None):
    n = hA.shape[0]
    pa, dt = _host_buf(hA, n, dtype)
    pq, _ = _host_buf(hQ, n, dt)
    pr, _ = _host_buf(hR, n, dt)
    info = ctypes.c_int64(0)
    _check(lib().qr_factor_host(n, s, dt, pa, n, pq, n, pr, n, ctypes.addressof(info)))
    return hQ, hR, info.value


# ----------------------------------------------------------------------- multi-GPU (block-cyclic)

def local_cols(n, s, nranks, rank):
    """Columns rank `rank` stores: panels p = rank, rank + nranks, ... of width s (the last ragged)."""
    return int(lib().sf_local_cols(n, s, nranks, rank))


def global_columns(n, s, nranks, rank):
    """Global column index of each local column of `rank` (block-cyclic by s-column panels)."""
    cols = []
    for p in range(rank, (n + s - 1) // s, nranks):
        cols.extend(range(p * s, min((p + 1) * s, n)))
    return cols


class Comm:
    """A libstepfact communicator: NCCL (one process per GPU) or loopback (all ranks here)."""

    def __init__(self, handle, nranks, local_ranks):
        self.handle = handle
        self.nranks = nranks
        self.local_ranks = local_ranks

    @classmethod
    def nccl(cls, nranks, rank, uid):
        h = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(uid))
        _check(lib().sf_comm_init(ctypes.byref(h), nranks, rank, buf))
        return cls(h, nranks, [rank])

    @classmethod
    def loopback(cls, nranks):
        h = ctypes.c_void_p()
        _check(lib().sf_comm_init_loopback(ctypes.byref(h), nranks))
        return cls(h, nranks, list(range(nranks)))

    def set_push(self, on=True):
        """Panel transport: device-initiated push (f3) instead of the broadcast (stepfact.h)."""
        _check(lib().sf_comm_set_push(self.handle, 1 if on else 0))

    def bcast_bytes(self):
        """Payload bytes of the panel messages this communicator has broadcast so far."""
        return int(lib().sf_comm_bcast_bytes(self.handle))

    def destroy(self):
        if self.handle is not None:
            _check(lib().sf_comm_destroy(self.handle))
            self.handle = None


def unique_id():
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().sf_get_unique_id(buf))
    return bytes(buf)


def _ptr_array(xs):
    arr = (ctypes.c_void_p * len(xs))()
    for i, x in enumerate(xs):
        arr[i] = None if x is None else (x.data_ptr() if hasattr(x, "data_ptr") else int(x))
    return arr


def chol_dist(comm, n, s, dA, dL, ld, d_info, dtype=None, stream=None):
    """chol_factor_dist: lists (one entry per local rank) of column-major local buffers."""
    dtype = _dt(dtype, *dA, *dL)
    _check(lib().chol_factor_dist(comm.handle, n, s, dtype, _ptr_array(dA), _ptr_array(dL), ld, _ptr_array(d_info),
                                  _stream(stream)))


def lu_dist(comm, n, s, dA, dLU, ld, d_info, dtype=None, stream=None):
    dtype = _dt(dtype, *dA, *dLU)
    _check(lib().lu_factor_dist(comm.handle, n, s, dtype, _ptr_array(dA), _ptr_array(dLU), ld, _ptr_array(d_info),
                                _stream(stream)))


def qr_dist(comm, n, s, dA, dQ, dR, ld, d_info, dtype=None, stream=None):
    dtype = _dt(dtype, *dA, *dQ, *dR)
    _check(lib().qr_factor_dist(comm.handle, n, s, dtype, _ptr_array(dA), _ptr_array(dQ), _ptr_array(dR), ld,
                                _ptr_array(d_info), _stream(stream)))


def scatter_cyclic(B, n, s, nranks, rank):
    """Local block-cyclic storage of `rank` from a column-major buffer B (torch, B[j] = column
    j): a (local_cols, n) tensor, i.e. column-major local columns with ld = n."""
    cols = global_columns(n, s, nranks, rank)
    return B[cols].contiguous()


def gather_cyclic(locals_, n, s, nranks, out):
    """Inverse of scatter_cyclic: write each rank's local columns into the column-major out."""
    for r, X in enumerate(locals_):
        cols = global_columns(n, s, nranks, r)
        if cols:
            out[cols] = X
    return out

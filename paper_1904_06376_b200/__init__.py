"""paper_1904_06376_b200 -- FP32 GEMM from BF16 tensor-core products on B200 (sm_100a).

Thin Python binding of ``libbf16x.so`` (C ABI in ``include/bf16x.h``): argument
marshalling only.  Every step of the method -- the split of P:180-184, the partial
products and bin sums of P:247-277/P:376-380, the promotion and the epilogue -- runs
in the CUDA kernels of ``csrc/``.  PyTorch is used for device memory and streams.
There is no CPU fallback: if the library or a B200 is missing, every call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BF16X_LIB") or os.path.join(_HERE, "libbf16x.so")   # BF16X_LIB: diagnostic builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "bf16x.h")

SUCCESS, ERR_CUDA, ERR_ALLOC, ERR_ARCH, ERR_SINGULAR, NOT_CONVERGED = 0, 1, 2, 3, 4, 5
ACC_IN, ACC_OUT = 1, 2
SCALED_PIECES, FP64_COMBINE, SPLIT_TRANSPOSED, NO_STREAM_K, A_PIECES_MN = 4, 8, 16, 32, 64   # bf16x.h flags
VARIANTS = (1, 3, 5, 6, 7, 8, 9)
PIECES = {1: 1, 3: 2, 6: 3, 8: 3, 9: 3}


class Bf16xError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class IRReport(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int), ("iterations", ctypes.c_int), ("info", ctypes.c_int),
                ("final_residual", ctypes.c_double), ("backward_error", ctypes.c_double),
                ("tol", ctypes.c_double), ("factor_ms", ctypes.c_double), ("refine_ms", ctypes.c_double),
                ("inner_iterations", ctypes.c_int)]


_lib = None
_i, _i64, _f, _d, _vp, _u = ctypes.c_int, ctypes.c_int64, ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_uint


def lib() -> ctypes.CDLL:
    """Load libbf16x.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `make lib` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        L.bf16x_split.argtypes = [_i64, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _vp]
        L.bf16x_split_t.argtypes = [_i64, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _vp]
        L.bf16x_split_ex.argtypes = [_i64, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _u, _vp]
        L.bf16x_split_operands.argtypes = [_i, _i, _i, _vp, _i64, _vp, _i64, _i, _vp, _i64, _i64, _vp, _i64, _i64, _vp]
        L.bf16x_split_operands_ex.argtypes = [_i, _i, _i, _vp, _i64, _vp, _i64, _i, _vp, _i64, _i64, _vp, _i64, _i64, _u,
                                              _vp]
        L.bf16x_gemm.argtypes = [_i, _i, _i, _f, _vp, _i, _vp, _i, _f, _vp, _i, _i]
        L.bf16x_gemm_workspace_size.argtypes = [_i, _i, _i, _i]
        L.bf16x_gemm_workspace_size.restype = ctypes.c_size_t
        L.bf16x_gemm_ex.argtypes = [_i, _i, _i, _f, _vp, _i, _vp, _i, _f, _vp, _i, _i, _u,
                                    _vp, _i64, _i64, _vp, _i64, _i64, _vp, _vp, ctypes.c_size_t, _vp]
        L.bf16x_gemm_cg.argtypes = [_i, _i, _i, _f, _vp, _i, _vp, _i, _f, _vp, _i, _i, _i, _vp]
        L.bf16x_gemm_host.argtypes = [_i, _i, _i, _f, _vp, _i, _vp, _i, _f, _vp, _i, _i]
        L.bf16x_gesv_ir.argtypes = [_i, _vp, _i, _vp, _vp, _i, _i, _d, _i, _vp, ctypes.POINTER(IRReport)]
        L.bf16x_gesv_gmres_ir.argtypes = [_i, _vp, _i, _vp, _vp, _i, _i, _i, _d, _d, _i, _vp,
                                          ctypes.POINTER(IRReport)]
        L.bf16x_getrf.argtypes = [_i, _vp, _i, _vp, _i, _i, ctypes.POINTER(ctypes.c_int)]
        L.bf16x_gesv16_batched.argtypes = [_i, _i, _vp, _i, _i64, _vp, _i64, _vp, _i64, _i, _i, _i, _vp, _vp, _vp,
                                           _vp, _vp]
        L.bf16x_set_stream.argtypes = [_vp]
        L.bf16x_get_stream.restype = _vp
        L.bf16x_status_string.argtypes = [_i]
        L.bf16x_status_string.restype = ctypes.c_char_p
        L.bf16x_launch_count.restype = ctypes.c_uint64
        L.bf16x_default_cta_group.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    if rc != SUCCESS:
        raise Bf16xError(rc, f"{what}: {lib().bf16x_status_string(rc).decode()}")


def _stream(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def _ptr(t) -> int:
    return int(t.data_ptr())


def device_check() -> None:
    _check(lib().bf16x_device_check(), "device_check")


def launch_count() -> int:
    """Kernels this process has launched through the library (all entry points)."""
    return int(lib().bf16x_launch_count())


def default_cta_group() -> int:
    """cta_group the library picks when none is forced (1: one CTA per SM, 128 x 256 tiles)."""
    return int(lib().bf16x_default_cta_group())


def release() -> None:
    lib().bf16x_release()


# ------------------------------------------------------------------------------------
# layout helpers: the ABI is column-major; torch tensors are usually row-major
# ------------------------------------------------------------------------------------
def _colmajor(t):
    """(ptr, rows, cols, ld) of a 2-D tensor viewed as a column-major matrix of t's shape,
    or None if its layout is not column-major."""
    if t.dim() != 2:
        raise ValueError("expected a 2-D tensor")
    r, c = t.shape
    if t.numel() == 0:
        return _ptr(t), r, c, max(1, r)
    if t.stride(0) == 1 and (c <= 1 or t.stride(1) >= max(1, r)):
        return _ptr(t), r, c, max(1, t.stride(1) if c > 1 else r)
    return None


def _rowmajor(t):
    """(ptr, rows, cols, ld) of t viewed as the column-major matrix t^T."""
    r, c = t.shape
    if t.numel() == 0:
        return _ptr(t), c, r, max(1, c)
    if t.stride(1) == 1 and (r <= 1 or t.stride(0) >= max(1, c)):
        return _ptr(t), c, r, max(1, t.stride(0) if r > 1 else c)
    return None


# ------------------------------------------------------------------------------------
# K1: split
# ------------------------------------------------------------------------------------
def split(x, pieces: int = 3, stream=None, scaled: bool = False):
    """b0, b1, b2 = (B16) pieces of an FP32 CUDA tensor (any 2-D strided layout with a unit
    stride, or 1-D contiguous).  Returns `pieces` uint16 tensors with x's shape and layout.
    scaled: the N2 power-of-two scaled pieces (b0, b1', b2') of DESIGN.md R29."""
    import torch
    if x.dtype != torch.float32 or not x.is_cuda:
        raise TypeError("split expects a float32 CUDA tensor")
    if x.numel() == 0:
        return tuple(torch.empty(x.shape, dtype=torch.uint16, device=x.device) for _ in range(pieces))
    if x.dim() == 1:
        x2 = x.reshape(-1, 1)
    else:
        x2 = x
    cm = _colmajor(x2)
    if cm is None:
        cm_rm = _rowmajor(x2)
        if cm_rm is None:
            x2 = x2.contiguous()
            cm_rm = _rowmajor(x2)
        ptr, rows, cols, ld = cm_rm
        outs = [torch.empty(x2.shape, dtype=torch.uint16, device=x.device) for _ in range(pieces)]
        ldp = max(1, rows)
    else:
        ptr, rows, cols, ld = cm
        outs = [torch.empty_strided(x2.shape, (1, max(1, rows)), dtype=torch.uint16, device=x.device)
                for _ in range(pieces)]
        ldp = max(1, rows)
    p = [_ptr(o) for o in outs] + [0] * (3 - pieces)
    if scaled:
        _check(lib().bf16x_split_ex(rows, cols, ptr, ld, p[0], p[1] or None, p[2] or None, ldp, SCALED_PIECES,
                                    _stream(stream)), "bf16x_split_ex")
    else:
        _check(lib().bf16x_split(rows, cols, ptr, ld, p[0], p[1] or None, p[2] or None, ldp, _stream(stream)),
               "bf16x_split")
    return tuple(o.reshape(x.shape) for o in outs)


def split_raw(rows, cols, x_ptr, ldx, p0, p1, p2, ldp, transpose=False, stream=None) -> None:
    fn = lib().bf16x_split_t if transpose else lib().bf16x_split
    _check(fn(rows, cols, x_ptr, ldx, p0, p1 or None, p2 or None, ldp, _stream(stream)),
           "bf16x_split_t" if transpose else "bf16x_split")


# ------------------------------------------------------------------------------------
# K2: GEMM
# ------------------------------------------------------------------------------------
def gemm_raw(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, variant=6, flags=0, A_pieces=None, ldap=0,
             a_plane=0, B_pieces=None, ldbp=0, b_plane=0, acc=None, stream=None) -> None:
    """Column-major bf16x_gemm_ex on raw device pointers (ints)."""
    _check(lib().bf16x_gemm_ex(m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, variant, flags,
                               A_pieces, ldap, a_plane, B_pieces, ldbp, b_plane, acc, None, 0, _stream(stream)),
           "bf16x_gemm_ex")


def gemm(A, B, C=None, alpha: float = 1.0, beta: float = 0.0, variant: int = 6, stream=None, cta_group: int = 0,
         scaled: bool = False, fp64_combine: bool = False, no_stream_k: bool = False):
    """C = alpha * A @ B + beta * C for FP32 CUDA tensors, computed with the bf16x`variant`
    split GEMM.  Column-major (Fortran) and row-major inputs are both used in place.
    scaled: N2 power-of-two scaled pieces (R29); fp64_combine: the paper's "d" variants (R30);
    no_stream_k: BF16X_NO_STREAM_K (each element independent of the problem's shape)."""
    import torch
    if variant not in VARIANTS:
        raise ValueError(f"variant must be one of {VARIANTS}")
    for t in (A, B):
        if t.dtype != torch.float32 or not t.is_cuda or t.dim() != 2:
            raise TypeError("gemm expects 2-D float32 CUDA tensors")
    m, k = A.shape
    k2, n = B.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    if C is None:
        if beta != 0.0:
            raise ValueError("beta != 0 needs C")
        if _colmajor(A) and _colmajor(B):
            C = torch.empty_strided((m, n), (1, max(1, m)), dtype=torch.float32, device=A.device)
        else:
            C = torch.empty((m, n), dtype=torch.float32, device=A.device)
    st = _stream(stream)
    a, b, c = _colmajor(A), _colmajor(B), _colmajor(C)
    if a and b and c:
        args = (m, n, k, alpha, a[0], a[3], b[0], b[3], beta, c[0], c[3], variant)
    else:
        a, b, c = _rowmajor(A), _rowmajor(B), _rowmajor(C)
        if not (a and b and c):
            raise ValueError("A, B, C must share one layout (all row-major or all column-major)")
        # row-major C = A B  <=>  column-major C^T = B^T A^T
        args = (n, m, k, alpha, b[0], b[3], a[0], a[3], beta, c[0], c[3], variant)
    flags = (SCALED_PIECES if scaled else 0) | (FP64_COMBINE if fp64_combine else 0) | (NO_STREAM_K if no_stream_k else 0)
    if cta_group and not flags:
        _check(lib().bf16x_gemm_cg(*args, cta_group, st), "bf16x_gemm_cg")
    else:
        _check(lib().bf16x_gemm_ex(*args, flags, None, 0, 0, None, 0, 0, None, None, 0, st), "bf16x_gemm_ex")
    return C


def gemm_host(A: np.ndarray, B: np.ndarray, C: np.ndarray | None = None, alpha=1.0, beta=0.0, variant=6):
    """bf16x_gemm_host on host (numpy, Fortran-ordered float32) buffers; returns C."""
    A = np.asfortranarray(A, dtype=np.float32)
    B = np.asfortranarray(B, dtype=np.float32)
    m, k = A.shape
    _, n = B.shape
    if C is None:
        C = np.zeros((m, n), dtype=np.float32, order="F")
    elif not (C.flags.f_contiguous and C.dtype == np.float32):
        raise ValueError("C must be a Fortran-ordered float32 array")
    _check(lib().bf16x_gemm_host(m, n, k, alpha, A.ctypes.data, max(1, m), B.ctypes.data, max(1, k), beta,
                                 C.ctypes.data, max(1, m), variant), "bf16x_gemm_host")
    return C


def gemm_host_ptr(m, n, k, alpha, A_ptr, lda, B_ptr, ldb, beta, C_ptr, ldc, variant=6) -> None:
    """bf16x_gemm_host on raw host pointers (e.g. pinned torch CPU tensors)."""
    _check(lib().bf16x_gemm_host(m, n, k, alpha, A_ptr, lda, B_ptr, ldb, beta, C_ptr, ldc, variant),
           "bf16x_gemm_host")


def workspace_size(m, n, k, variant) -> int:
    return int(lib().bf16x_gemm_workspace_size(m, n, k, variant))


# ------------------------------------------------------------------------------------
# LU + iterative refinement
# ------------------------------------------------------------------------------------
def gesv_ir(A, b, variant: int = 3, nb: int = 256, max_iter: int = 30, tol: float = 0.0):
    """Solve A x = b (A: n x n float32 CUDA, column-major or row-major -- row-major is
    transposed on the device first; b: float64 CUDA vector).  tol > 0: stop when
    ||r||_inf <= tol ||b||_inf (the paper's cond(A)*eps); 0: the R14 default.
    Returns (x, report, history)."""
    import torch
    n = A.shape[0]
    cm = _colmajor(A)
    if cm is None:
        A = A.t().contiguous().t()
        cm = _colmajor(A)
    x = torch.empty(n, dtype=torch.float64, device=A.device)
    b = b.to(torch.float64).contiguous()
    hist = np.zeros(max(1, max_iter) + 1, dtype=np.float64)
    rep = IRReport()
    rc = lib().bf16x_gesv_ir(n, cm[0], cm[3], _ptr(b), _ptr(x), variant, nb, float(tol), max_iter, hist.ctypes.data,
                             ctypes.byref(rep))
    if rc not in (SUCCESS, NOT_CONVERGED, ERR_SINGULAR):
        _check(rc, "bf16x_gesv_ir")
    return x, rep, hist[: rep.iterations + 1]


def _square_colmajor(A):
    cm = _colmajor(A)
    if cm is None:
        A = A.t().contiguous().t()
        cm = _colmajor(A)
    return A, cm


def gesv_gmres_ir(A, b, variant: int = 3, nb: int = 256, restart: int = 200, inner_tol: float = 1e-10,
                  max_iter: int = 30, tol: float = 0.0):
    """GMRES-IR (bf16x_gesv_gmres_ir): LU with bf16x trailing updates as the preconditioner of
    FP64 GMRES corrections.  Arguments as gesv_ir plus restart / inner_tol.
    Returns (x, report, history); report.inner_iterations = total Arnoldi steps."""
    import torch
    n = A.shape[0]
    A, cm = _square_colmajor(A)
    x = torch.empty(n, dtype=torch.float64, device=A.device)
    b = b.to(torch.float64).contiguous()
    hist = np.zeros(max(1, max_iter) + 1, dtype=np.float64)
    rep = IRReport()
    rc = lib().bf16x_gesv_gmres_ir(n, cm[0], cm[3], _ptr(b), _ptr(x), variant, nb, restart, float(inner_tol), float(tol),
                                   max_iter, hist.ctypes.data, ctypes.byref(rep))
    if rc not in (SUCCESS, NOT_CONVERGED, ERR_SINGULAR):
        _check(rc, "bf16x_gesv_gmres_ir")
    return x, rep, hist[: rep.iterations + 1]


def getrf(A, variant: int = 3, nb: int = 256):
    """P A = L U of a square float32 CUDA matrix (bf16x_getrf).  Returns (LU, ipiv, info):
    LU a column-major float32 CUDA tensor (a copy; A is not modified), ipiv int32 CUDA
    (0-based interchange sequence), info the 1-based first zero-pivot column or 0."""
    import torch
    n = A.shape[0]
    LU = torch.empty_strided((n, n), (1, max(1, n)), dtype=torch.float32, device=A.device)
    LU.copy_(A)
    cm = _colmajor(LU)
    ipiv = torch.zeros(max(1, n), dtype=torch.int32, device=A.device)
    info = ctypes.c_int(0)
    rc = lib().bf16x_getrf(n, cm[0], cm[3], _ptr(ipiv), variant, nb, ctypes.byref(info))
    if rc not in (SUCCESS, ERR_SINGULAR):
        _check(rc, "bf16x_getrf")
    return LU, ipiv[:n], int(info.value)


FORMATS16 = {"fp32": 0, "bf16": 1, "fp16": 2}


def gesv16_batched(A, b, tol, fmt: str = "bf16", pivot: bool = True, max_iter: int = 100, stream=None):
    """bf16x_gesv16_batched on CUDA tensors: A (batch, n, n) float32 (A[s] is system s, any
    layout: copied column-major), b (batch, n) float64, tol (batch,) float64.
    Returns (x (batch, n) float64, converged, iterations, info) as CUDA tensors."""
    import torch
    batch, n, _ = A.shape
    Acm = A.transpose(1, 2).contiguous()            # column-major per system, lda = n
    b = b.to(torch.float64).contiguous()
    tol = tol.to(torch.float64).contiguous()
    x = torch.empty(batch, n, dtype=torch.float64, device=A.device)
    conv = torch.empty(batch, dtype=torch.int32, device=A.device)
    its = torch.empty_like(conv)
    info = torch.empty_like(conv)
    st = _stream(stream)
    _check(lib().bf16x_gesv16_batched(n, batch, _ptr(Acm), max(1, n), n * n, _ptr(b), n, _ptr(x), n,
                                      FORMATS16[fmt], int(bool(pivot)), max_iter, _ptr(tol), _ptr(conv), _ptr(its),
                                      _ptr(info), st), "bf16x_gesv16_batched")
    return x, conv, its, info

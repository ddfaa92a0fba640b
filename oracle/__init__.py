"""CPU oracle for the BF16-split FP32 GEMM of arXiv 1904.06376 -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product package
(``paper_1904_06376_b200``) never imports it and shares no code with it.

The arithmetic lives in ``bf16x_oracle.c`` (plain C99, one IEEE FP32 operation
per source operation, no FTZ); this module is argument marshalling plus the
plain-numpy error metrics and the iterative-refinement loop (§III), each
citing the passage it follows.  Pins: ``tests/test_oracle_*.py``; see DESIGN.md
"Oracle pins" for the list (the LU-IR and GMRES-IR convergence statistics are
*parity unpinned*: the paper's tables are for single-BF16/FP16 LU; GMRES
itself is pinned by Krylov theory and brute-force least squares, test_oracle_gmres.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="F_CONTIGUOUS")
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain gcc, see Makefile flags)."""
    src = os.path.join(_HERE, "bf16x_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-C", os.path.dirname(_HERE), "oracle"])
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_bf16_round.argtypes = [ctypes.c_float]
        L.orc_bf16_round.restype = ctypes.c_uint16
        L.orc_bf16_widen.argtypes = [ctypes.c_uint16]
        L.orc_bf16_widen.restype = ctypes.c_float
        L.orc_split.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp]
        L.orc_split_patterns.argtypes = [ctypes.c_uint64, ctypes.c_int64, _vp, _vp, _vp]
        L.orc_partials.argtypes = [ctypes.c_int] * 3 + [_vp, ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_int, _vp]
        L.orc_gemm_split_cols.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_float, _vp, ctypes.c_int, _vp, ctypes.c_int,
                                          ctypes.c_float, _vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp])
        L.orc_split_scaled.argtypes = [ctypes.c_int64, _vp, _vp, _vp, _vp]
        L.orc_split_scaled_patterns.argtypes = [ctypes.c_uint64, ctypes.c_int64, _vp, _vp, _vp]
        L.orc_gemm_split_ex_cols.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_float, _vp, ctypes.c_int, _vp, ctypes.c_int,
                                             ctypes.c_float, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp,
                                             ctypes.c_int, _vp])
        L.orc_gemm_split.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_float, _vp, ctypes.c_int, _vp, ctypes.c_int,
                                     ctypes.c_float, _vp, ctypes.c_int, ctypes.c_int])
        L.orc_sgemm_fma_cols.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_float, _vp, ctypes.c_int, _vp, ctypes.c_int,
                                         ctypes.c_float, _vp, ctypes.c_int, _vp, ctypes.c_int, _vp])
        L.orc_dgemm_cols.argtypes = [ctypes.c_int] * 3 + [_vp, ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_int, _vp]
        L.orc_getrf_split.argtypes = [ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int]
        L.orc_lu_solve_f64.argtypes = [ctypes.c_int, _vp, ctypes.c_int, _vp, _vp]
        L.orc_residual_f64.argtypes = [ctypes.c_int, _vp, ctypes.c_int, _vp, _vp, _vp]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_fp16_round.argtypes = [ctypes.c_float]
        L.orc_fp16_round.restype = ctypes.c_uint16
        L.orc_fp16_widen.argtypes = [ctypes.c_uint16]
        L.orc_fp16_widen.restype = ctypes.c_float
        L.orc_getrf16.argtypes = [ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _colmajor_f32(x) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    if x.ndim == 1:
        x = x.reshape(-1, 1)
    return np.asfortranarray(x)


def num_threads() -> int:
    return int(lib().orc_num_threads())


# --------------------------------------------------------------------------
# O-1 / O-2: conversion and split (§II-A)
# --------------------------------------------------------------------------
def bf16_round(x: float) -> int:
    """(B16) operator on one FP32 value -> 16-bit pattern (R1/R3/R4)."""
    return int(lib().orc_bf16_round(ctypes.c_float(float(np.float32(x)))))


def bf16_widen(b: int) -> float:
    """(F32) widening of a 16-bit pattern (exact)."""
    return float(lib().orc_bf16_widen(ctypes.c_uint16(b)))


def split(x) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """3-way split of FP32 values.  Returns three uint16 arrays of x's shape."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    flat = x.reshape(-1)
    out = [np.empty(flat.shape, dtype=np.uint16) for _ in range(3)]
    lib().orc_split(flat.size, _ptr(flat), _ptr(out[0]), _ptr(out[1]), _ptr(out[2]))
    return tuple(o.reshape(x.shape) for o in out)


def split_patterns(first: int, count: int):
    """Split every FP32 bit pattern in [first, first+count)."""
    out = [np.empty(count, dtype=np.uint16) for _ in range(3)]
    lib().orc_split_patterns(first, count, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]))
    return tuple(out)


def split_scaled(x) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """N2 scaled split (R29): b0, b1' = (B16)(2^8 (x - b0)), b2' = (B16)(2^8 (2^8 (x - b0) - b1')).

    x = b0 + 2^-8 b1' + 2^-16 b2' for every finite x (pinned in test_oracle_scaled.py)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    flat = x.reshape(-1)
    out = [np.empty(flat.shape, dtype=np.uint16) for _ in range(3)]
    lib().orc_split_scaled(flat.size, _ptr(flat), _ptr(out[0]), _ptr(out[1]), _ptr(out[2]))
    return tuple(o.reshape(x.shape) for o in out)


def split_scaled_patterns(first: int, count: int):
    """Scaled split (R29) of every FP32 bit pattern in [first, first+count)."""
    out = [np.empty(count, dtype=np.uint16) for _ in range(3)]
    lib().orc_split_scaled_patterns(first, count, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]))
    return tuple(out)


def widen(p: np.ndarray) -> np.ndarray:
    """Exact BF16 pattern -> FP32 values (bits << 16); plain numpy bit view."""
    return (np.asarray(p, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


# --------------------------------------------------------------------------
# O-3..O-6: partial products, combine, scale, FP32/FP64 references
# --------------------------------------------------------------------------
def partials(A, B, cols=None) -> np.ndarray:
    """All nine Z^(i,j) for C = A*B; returns array [3,3,m,ncols]."""
    A = _colmajor_f32(A)
    B = _colmajor_f32(B)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    cols_arr = np.arange(n, dtype=np.int32) if cols is None else np.ascontiguousarray(cols, dtype=np.int32)
    nc = cols_arr.size
    Z = np.zeros((9, nc, m), dtype=np.float32)
    lib().orc_partials(m, n, k, _ptr(A), max(1, m), _ptr(B), max(1, k), _ptr(cols_arr), nc, _ptr(Z))
    return Z.reshape(3, 3, nc, m).transpose(0, 1, 3, 2)


def gemm(A, B, C=None, alpha=1.0, beta=0.0, variant=6, cols=None, scaled=False, fp64_combine=False) -> np.ndarray:
    """Split GEMM C_out = alpha*A*B + beta*C (BLAS scaling R19).

    variant in {1, 3, 5, 6, 7, 8, 9}.  scaled: N2 power-of-two scaled pieces (R29);
    fp64_combine: the paper's "d" variants, bins collected in FP64 and rounded once
    (R30).  Returns the m x len(cols) FP32 result."""
    A = _colmajor_f32(A)
    B = _colmajor_f32(B)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    cols_arr = np.arange(n, dtype=np.int32) if cols is None else np.ascontiguousarray(cols, dtype=np.int32)
    nc = cols_arr.size
    out = np.zeros((m, nc), dtype=np.float32, order="F")
    if C is None:
        Cin = np.zeros((1, 1), dtype=np.float32, order="F")
        ldc = max(1, m)
        if beta != 0.0:
            raise ValueError("beta != 0 needs C")
    else:
        Cin = _colmajor_f32(C)
        ldc = max(1, m)
    mode = (1 if scaled else 0) | (2 if fp64_combine else 0)
    rc = lib().orc_gemm_split_ex_cols(m, n, k, float(alpha), _ptr(A), max(1, m), _ptr(B), max(1, k), float(beta),
                                      _ptr(Cin), ldc, int(variant), mode, _ptr(cols_arr), nc, _ptr(out))
    if rc != 0:
        raise ValueError(f"oracle gemm returned {rc}")
    return out


def sgemm_fma(A, B, C=None, alpha=1.0, beta=0.0, cols=None) -> np.ndarray:
    """FP32 FMA reference GEMM (§II-C)."""
    A = _colmajor_f32(A)
    B = _colmajor_f32(B)
    m, k = A.shape
    _, n = B.shape
    cols_arr = np.arange(n, dtype=np.int32) if cols is None else np.ascontiguousarray(cols, dtype=np.int32)
    nc = cols_arr.size
    out = np.zeros((m, nc), dtype=np.float32, order="F")
    Cin = np.zeros((1, 1), dtype=np.float32, order="F") if C is None else _colmajor_f32(C)
    lib().orc_sgemm_fma_cols(m, n, k, float(alpha), _ptr(A), max(1, m), _ptr(B), max(1, k), float(beta),
                             _ptr(Cin), max(1, m), _ptr(cols_arr), nc, _ptr(out))
    return out


def dgemm(A, B, cols=None) -> np.ndarray:
    """FP64 reference product of FP32 data ("DGEMM"), sequential FP64 sums."""
    A = _colmajor_f32(A)
    B = _colmajor_f32(B)
    m, k = A.shape
    _, n = B.shape
    cols_arr = np.arange(n, dtype=np.int32) if cols is None else np.ascontiguousarray(cols, dtype=np.int32)
    nc = cols_arr.size
    out = np.zeros((m, nc), dtype=np.float64, order="F")
    lib().orc_dgemm_cols(m, n, k, _ptr(A), max(1, m), _ptr(B), max(1, k), _ptr(cols_arr), nc, _ptr(out))
    return out


# --------------------------------------------------------------------------
# Metrics (north star; Fig. 2 caption)
# --------------------------------------------------------------------------
def normwise_error(C, C64, A, B) -> float:
    """North-star metric ||C - C64||_F / (||A||_F ||B||_F), in FP64."""
    C = np.asarray(C, dtype=np.float64)
    C64 = np.asarray(C64, dtype=np.float64)
    den = np.linalg.norm(np.asarray(A, dtype=np.float64)) * np.linalg.norm(np.asarray(B, dtype=np.float64))
    return float(np.linalg.norm(C - C64) / den) if den > 0 else float(np.linalg.norm(C - C64))


def relative_frobenius_error(C, C64) -> float:
    """The paper's ||C - DGEMM||_F / ||DGEMM||_F (Fig. 2 caption)."""
    C64 = np.asarray(C64, dtype=np.float64)
    return float(np.linalg.norm(np.asarray(C, dtype=np.float64) - C64) / np.linalg.norm(C64))


# --------------------------------------------------------------------------
# O-7: LU + iterative refinement (§III)
# --------------------------------------------------------------------------
def getrf(A, variant=3, nb=64):
    """Blocked LU, FP32 panel, split-GEMM trailing update.  Returns (LU, ipiv, info)."""
    LU = np.array(A, dtype=np.float32, order="F", copy=True)
    n = LU.shape[0]
    ipiv = np.zeros(n, dtype=np.int32)
    info = lib().orc_getrf_split(n, _ptr(LU), max(1, n), _ptr(ipiv), int(nb), int(variant))
    return LU, ipiv, int(info)


def lu_solve_f64(LU, ipiv, b) -> np.ndarray:
    """FP64 forward/back substitution with the FP32 factors."""
    n = LU.shape[0]
    x = np.array(b, dtype=np.float64, copy=True)
    lib().orc_lu_solve_f64(n, _ptr(LU), max(1, n), _ptr(ipiv), _ptr(x))
    return x


def residual_f64(A, b, x) -> np.ndarray:
    A = _colmajor_f32(A)
    n = A.shape[0]
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    r = np.empty(n, dtype=np.float64)
    lib().orc_residual_f64(n, _ptr(A), max(1, n), _ptr(b), _ptr(x), _ptr(r))
    return r


def gesv_ir(A, b, variant=3, nb=64, max_iter=30, tol=0.0):
    """LU + iterative refinement: factor in low precision; loop { r = b - A x
    in FP64; solve A d = r with the factors in FP64; x += d }.

    Stopping rule (reading R14): with tol > 0 converged when
    ||r||_inf <= tol * ||b||_inf ("a residual tolerance of cond(A)*eps": tol =
    cond(A) * 2^-53); otherwise when ||r||_inf <= sqrt(n) * ||x||_inf * ||A||_inf * 2^-53
    (LAPACK dsgesv's rule); stagnation = residual not halved over 3 consecutive iterations.
    Returns dict(x, converged, iterations, info, history)."""
    A = _colmajor_f32(A)
    n = A.shape[0]
    LU, ipiv, info = getrf(A, variant=variant, nb=nb)
    if info != 0:
        return dict(x=np.zeros(n), converged=False, iterations=0, info=info, history=[])
    anrm = float(np.max(np.sum(np.abs(A.astype(np.float64)), axis=1)))
    bnrm = float(np.max(np.abs(np.asarray(b, dtype=np.float64)))) if n else 0.0
    eps = 2.0 ** -53
    x = lu_solve_f64(LU, ipiv, b)
    hist = []
    converged = False
    it = 0
    for it in range(0, max_iter + 1):
        r = residual_f64(A, b, x)
        rn = float(np.max(np.abs(r)))
        hist.append(rn)
        thr = tol * bnrm if tol > 0 else np.sqrt(n) * float(np.max(np.abs(x))) * anrm * eps
        if rn <= thr:
            converged = True
            break
        if it == max_iter:
            break
        if len(hist) >= 4 and hist[-1] > 0.5 * hist[-4]:
            break
        x = x + lu_solve_f64(LU, ipiv, r)
    return dict(x=x, converged=converged, iterations=it, info=0, history=hist)


# --------------------------------------------------------------------------
# O-8: GMRES and GMRES-IR (§III "combining Iterative Refinement with an
# Iterative Solver like GMRES [iterativerefinement-fp16][templates]"
# §IV-B "apply GMRES instead of iterative refinement, and use the LU decomposition
# in the lower precision ... as a pre-conditioner")
# --------------------------------------------------------------------------
def gmres(matvec, psolve, b, x0=None, restart=None, tol=1e-10, max_cycles=1):
    """Left-preconditioned restarted GMRES(m) in FP64, step by step as in the paper's
    cited GMRES template (Barrett et al., "Templates for the Solution of Linear Systems",
    section 2.3.4): Arnoldi with modified Gram-Schmidt on M^-1 A, Givens rotations on the
    Hessenberg column, least-squares update x += V y at the end of each cycle.

    Solves M^-1 A x = M^-1 b.  matvec(v) = A v, psolve(v) = M^-1 v (both FP64).  A cycle
    ends after `restart` Arnoldi steps, on an exact breakdown (h_{j+1,j} == 0: the
    Krylov space is invariant, the least-squares solution is exact), or when the rotated
    residual |s_{j+1}| <= tol * ||M^-1 (b - A x0)||_2 (reading R25).
    Returns dict(x, iterations = Arnoldi steps, history = [|s_{j+1}|], converged)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    m = n if restart is None else max(1, min(int(restart), n))
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    r = psolve(b - matvec(x))
    beta0 = float(np.linalg.norm(r))
    hist = []
    steps = 0
    if beta0 == 0.0:
        return dict(x=x, iterations=0, history=[0.0], converged=True)
    converged = False
    for _cycle in range(max_cycles):
        beta = float(np.linalg.norm(r))
        V = np.zeros((n, m + 1))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        s = np.zeros(m + 1)
        s[0] = beta
        V[:, 0] = r / beta
        jm = 0
        for j in range(m):
            w = psolve(matvec(V[:, j]))
            for i in range(j + 1):                      # modified Gram-Schmidt
                H[i, j] = float(w @ V[:, i])
                w = w - H[i, j] * V[:, i]
            hnext = float(np.linalg.norm(w))
            H[j + 1, j] = hnext
            if hnext != 0.0:
                V[:, j + 1] = w / hnext
            for i in range(j):                          # previous rotations on column j
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = float(np.hypot(H[j, j], H[j + 1, j]))  # new rotation annihilates H[j+1, j]
            cs[j] = H[j, j] / d
            sn[j] = H[j + 1, j] / d
            H[j, j] = d
            H[j + 1, j] = 0.0
            s[j + 1] = -sn[j] * s[j]
            s[j] = cs[j] * s[j]
            steps += 1
            jm = j + 1
            hist.append(abs(float(s[j + 1])))
            if abs(s[j + 1]) <= tol * beta0 or hnext == 0.0:
                converged = True
                break
        y = np.zeros(jm)                                 # back substitution H y = s
        for i in range(jm - 1, -1, -1):
            y[i] = (s[i] - H[i, i + 1:jm] @ y[i + 1:jm]) / H[i, i]
        x = x + V[:, :jm] @ y
        if converged:
            break
        r = psolve(b - matvec(x))
    return dict(x=x, iterations=steps, history=hist, converged=converged)


def gmres_ir(A, b, variant=3, nb=64, restart=200, inner_tol=1e-10, max_iter=30, tol=0.0):
    """GMRES-IR: factor once in low precision (getrf, the split-GEMM trailing updates of
    P:406); outer loop as gesv_ir (r = b - A x in FP64, same stopping and stagnation rules,
    R14), but the correction equation A d = r is solved by one cycle of FP64 GMRES left-
    preconditioned with the low-precision factors (reading R25), x0 = 0.
    Returns dict(x, converged, iterations = outer corrections, inner_iterations = total
    Arnoldi steps, info, history)."""
    A = _colmajor_f32(A)
    n = A.shape[0]
    LU, ipiv, info = getrf(A, variant=variant, nb=nb)
    if info != 0:
        return dict(x=np.zeros(n), converged=False, iterations=0, inner_iterations=0, info=info, history=[])
    anrm = float(np.max(np.sum(np.abs(A.astype(np.float64)), axis=1)))
    bnrm = float(np.max(np.abs(np.asarray(b, dtype=np.float64)))) if n else 0.0
    eps = 2.0 ** -53
    zero = np.zeros(n)
    matvec = lambda v: -residual_f64(A, zero, v)          # A v, FP64 sums of FP32 A
    psolve = lambda v: lu_solve_f64(LU, ipiv, v)
    x = np.zeros(n)
    hist = []
    converged = False
    inner = 0
    it = 0
    for it in range(0, max_iter + 1):
        r = residual_f64(A, b, x)
        rn = float(np.max(np.abs(r)))
        hist.append(rn)
        thr = tol * bnrm if tol > 0 else np.sqrt(n) * float(np.max(np.abs(x))) * anrm * eps
        if rn <= thr:
            converged = True
            break
        if it == max_iter:
            break
        if len(hist) >= 4 and hist[-1] > 0.5 * hist[-4]:
            break
        g = gmres(matvec, psolve, r, restart=restart, tol=inner_tol, max_cycles=1)
        inner += g["iterations"]
        x = x + g["x"]
    return dict(x=x, converged=converged, iterations=it, inner_iterations=inner, info=0, history=hist)


# --------------------------------------------------------------------------
# O-9: the Fig. 5 SGETRF accuracy measure (§IV-A: "SGETRF vs BFLOAT16x3_6 LU
# Decomposition: Element errors average improvement ... The comparison points were results
# from DGETRF on the same input data")
# --------------------------------------------------------------------------
def lu_nopivot_f64(M) -> np.ndarray:
    """Right-looking LU without pivoting in FP64 (the textbook elimination), L unit lower and
    U packed in one array.  Applied to P A with the pivots of the factorisation under test, it
    is the FP64 (DGETRF) factorisation that factorisation approximates element by element."""
    M = np.array(M, dtype=np.float64, copy=True)
    n = M.shape[0]
    for j in range(n):
        M[j + 1:, j] /= M[j, j]
        M[j + 1:, j + 1:] -= np.outer(M[j + 1:, j], M[j, j + 1:])
    return M


def row_permutation(ipiv) -> np.ndarray:
    """p such that (P A) = A[p]: the LAPACK interchange sequence applied in order."""
    ipiv = np.asarray(ipiv)
    p = np.arange(ipiv.size)
    for j, q in enumerate(ipiv):
        p[[j, q]] = p[[q, j]]
    return p


def lu_element_error(A, LU, ipiv) -> float:
    """Mean over all entries of |LU - D| / |D|, D = FP64 LU of P A with the same pivots (R26)."""
    A = np.asarray(A, dtype=np.float64)
    D = lu_nopivot_f64(A[row_permutation(ipiv)])
    den = np.abs(D)
    mask = den > 0
    return float(np.mean(np.abs(np.asarray(LU, dtype=np.float64)[mask] - D[mask]) / den[mask]))


# --------------------------------------------------------------------------
# O-10: fully 16-bit LU and its refinement (N4; §IV-B, reading R28)
# --------------------------------------------------------------------------
FORMATS = {"fp32": 0, "bf16": 1, "fp16": 2}


def fp16_round(x: float) -> int:
    """IEEE binary16 RNE of one FP32 value -> 16-bit pattern (overflow -> Inf, subnormals kept)."""
    return int(lib().orc_fp16_round(ctypes.c_float(float(np.float32(x)))))


def fp16_widen(h: int) -> float:
    return float(lib().orc_fp16_widen(ctypes.c_uint16(h)))


def getrf16(A, fmt="bf16", pivot=True):
    """Gaussian elimination with every stored result rounded to the working format.
    Returns (LU, ipiv, info); LU holds format values (widened to FP32)."""
    LU = np.array(A, dtype=np.float32, order="F", copy=True)
    n = LU.shape[0]
    ipiv = np.zeros(n, dtype=np.int32)
    info = lib().orc_getrf16(n, _ptr(LU), max(1, n), _ptr(ipiv), FORMATS[fmt], int(bool(pivot)))
    return LU, ipiv, int(info)


def norm2_seq(v) -> float:
    """||v||_2 as a plain sequential FP64 sum of squares (fixed order, reproducible)."""
    s = 0.0
    for t in np.asarray(v, dtype=np.float64):
        s += float(t) * float(t)
    return float(np.sqrt(s))


def gesv16_ir(A, b, fmt="bf16", pivot=True, tol=None, max_iter=100):
    """The §IV-B refinement experiment: factor in the working format, then loop
    { r = b - A x in FP64; x += U^-1 L^-1 P r in FP64 } from x0 = U^-1 L^-1 P b, converged
    when ||r||_2 <= tol ||b||_2 with tol = cond(A) * 2^-53 ("a residual tolerance of
    cond(A)*eps"; the caller passes cond(A)*2^-53).  Returns dict(x, converged,
    iterations = corrections applied, info)."""
    A = _colmajor_f32(A)
    n = A.shape[0]
    b = np.ascontiguousarray(b, dtype=np.float64)
    LU, ipiv, info = getrf16(A, fmt=fmt, pivot=pivot)
    if info != 0:
        return dict(x=np.zeros(n), converged=False, iterations=0, info=info)
    nb = norm2_seq(b)
    x = lu_solve_f64(LU, ipiv, b)
    for it in range(max_iter + 1):
        r = residual_f64(A, b, x)
        if norm2_seq(r) <= tol * nb:
            return dict(x=x, converged=True, iterations=it, info=0)
        if it == max_iter or not np.all(np.isfinite(x)):
            break
        x = x + lu_solve_f64(LU, ipiv, r)
    return dict(x=x, converged=False, iterations=it, info=0)

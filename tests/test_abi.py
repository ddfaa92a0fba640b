"""The C ABI boundary: libbf16x.so loads, exports every entry point include/bf16x.h declares,
validates arguments LAPACK-style on the host, and (without a GPU) refuses to compute instead of
falling back to the CPU."""
import ctypes
import re

import pytest

import paper_1904_06376_b200 as bx


def _declared_functions():
    src = open(bx.HEADER_PATH).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(bf16x_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = bx.lib()
    names = _declared_functions()
    assert {"bf16x_split", "bf16x_split_t", "bf16x_gemm", "bf16x_gemm_ex", "bf16x_gemm_host",
            "bf16x_gesv_ir", "bf16x_gemm_workspace_size"} <= set(names)
    for name in names:
        assert hasattr(L, name), name


def test_gemm_argument_errors():
    L = bx.lib()
    f = L.bf16x_gemm
    assert f(-1, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6) == -1
    assert f(4, -1, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6) == -2
    assert f(4, 4, -1, 1.0, None, 4, None, 4, 0.0, None, 4, 6) == -3
    assert f(4, 4, 4, 1.0, None, 3, None, 4, 0.0, None, 4, 6) == -6
    assert f(4, 4, 4, 1.0, None, 4, None, 3, 0.0, None, 4, 6) == -8
    assert f(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 3, 6) == -11
    assert f(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 4) == -12
    ex = L.bf16x_gemm_ex
    assert ex(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6, 128, None, 0, 0, None, 0, 0, None, None, 0, None) == -13
    # FP64 combine (R30) excludes the accumulator carry and the one-product variant
    assert ex(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6, 9, None, 0, 0, None, 0, 0, 16, None, 0, None) == -13
    assert ex(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 1, 8, None, 0, 0, None, 0, 0, None, None, 0, None) == -13
    assert ex(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6, 0, 16, 3, 32, None, 0, 0, None, None, 0, None) == -14
    assert ex(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6, 0, None, 0, 0, 16, 8, 4, None, None, 0, None) == -16
    assert ex(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6, 1, None, 0, 0, None, 0, 0, None, None, 0, None) == -19
    # BF16X_A_PIECES_MN (64): A's pieces in A's own layout, ldap >= m, a_plane >= ldap * k, both % 8
    mn = bx.A_PIECES_MN
    assert ex(12, 4, 4, 1.0, None, 12, None, 4, 0.0, None, 12, 6, mn, 16, 8, 64, None, 0, 0, None, None, 0, None) == -14
    assert ex(4, 4, 12, 1.0, None, 4, None, 12, 0.0, None, 4, 6, mn, 16, 8, 88, None, 0, 0, None, None, 0, None) == -14
    assert ex(4, 4, 12, 1.0, None, 4, None, 12, 0.0, None, 4, 6, mn, 16, 12, 144, None, 0, 0, None, None, 0, None) == -14
    # (valid MN layout: the host checks pass and the call stops at the device check, not computing on the CPU)
    assert ex(4, 4, 12, 1.0, None, 4, None, 12, 0.0, None, 4, 6, mn, 16, 8, 96, None, 0, 0, None, None, 0, None) in (
        bx.ERR_ARCH, bx.ERR_CUDA)


def test_split_operands_ex_argument_errors():
    so = bx.lib().bf16x_split_operands_ex
    mn = bx.A_PIECES_MN
    # MN layout of A's pieces: ldap >= m, a_plane >= ldap * k (-9); B as bf16x_split_operands (-12)
    assert so(12, 4, 4, None, 12, None, 4, 3, 16, 8, 64, 16, 8, 64, mn, None) == -9
    assert so(4, 4, 12, None, 4, None, 12, 3, 16, 8, 88, 16, 16, 64, mn, None) == -9
    assert so(4, 4, 12, None, 4, None, 12, 3, 16, 8, 96, 16, 8, 64, mn, None) == -12
    assert so(4, 4, 12, None, 4, None, 12, 3, 16, 8, 96, 16, 16, 64, 128, None) == -13
    assert so(4, 4, 12, None, 4, None, 12, 4, 16, 8, 96, 16, 16, 64, mn, None) == -8
    # K-major A (no flag): ldap >= k, a_plane >= ldap * m
    assert so(4, 4, 12, None, 4, None, 12, 3, 16, 8, 96, 16, 16, 64, 0, None) == -9
    assert so(4, 4, 12, None, 4, None, 12, 3, 16, 16, 64, 16, 16, 64, 0, None) in (bx.ERR_ARCH, bx.ERR_CUDA)


def test_split_argument_errors():
    L = bx.lib()
    s = L.bf16x_split
    assert s(-1, 2, None, 1, 16, None, None, 1, None) == -1
    assert s(2, -1, None, 2, 16, None, None, 2, None) == -2
    assert s(4, 2, None, 3, 16, None, None, 4, None) == -4
    assert s(4, 2, None, 4, None, None, None, 4, None) == -5
    assert s(4, 2, None, 4, 16, None, 32, 4, None) == -7
    assert s(4, 2, None, 4, 16, None, None, 3, None) == -8
    assert L.bf16x_split_t(4, 6, None, 4, 16, None, None, 5, None) == -8
    se = L.bf16x_split_ex
    se.argtypes = [ctypes.c_int64] * 2 + [ctypes.c_void_p, ctypes.c_int64] + [ctypes.c_void_p] * 3 + \
        [ctypes.c_int64, ctypes.c_uint, ctypes.c_void_p]
    assert se(4, 2, None, 4, 16, None, None, 4, 64, None) == -9          # unknown flag
    assert se(4, 6, None, 4, 16, None, None, 5, 4 | 16, None) == -8      # transposed: ldp >= cols


def test_workspace_size_formula():
    # 2 bytes * p pieces * (round_up(m, 8) + n) rows * round_up(k, 8) (A's pieces keep A's layout, ld round_up(m, 8))
    assert bx.workspace_size(100, 50, 33, 6) == 2 * 3 * 154 * 40
    assert bx.workspace_size(100, 50, 33, 3) == 2 * 2 * 154 * 40
    assert bx.workspace_size(100, 50, 33, 5) == 2 * (2 * 104 + 3 * 50) * 40
    assert bx.workspace_size(96, 50, 33, 6) == 2 * 3 * 146 * 40


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = bx.lib()
    rc = L.bf16x_gemm(4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 6)
    assert rc == bx.ERR_ARCH
    assert b"sm_100" in L.bf16x_status_string(rc)


def test_solver_argument_errors():
    L = bx.lib()
    rep = bx.IRReport()
    g = L.bf16x_gesv_gmres_ir
    assert g(-1, None, 1, None, None, 3, 0, 0, 0.0, 0.0, 0, None, ctypes.byref(rep)) == -1
    assert g(4, None, 3, None, None, 3, 0, 0, 0.0, 0.0, 0, None, ctypes.byref(rep)) == -3
    assert g(4, None, 4, None, None, 7, 0, 0, 0.0, 0.0, 0, None, ctypes.byref(rep)) == -6
    assert g(4, None, 4, None, None, 3, 0, 0, -1.0, 0.0, 0, None, ctypes.byref(rep)) == -9
    assert g(4, None, 4, None, None, 3, 0, 0, 0.0, float("nan"), 0, None, ctypes.byref(rep)) == -10
    assert g(4, None, 4, None, None, 3, 0, 0, 0.0, 0.0, 0, None, None) == -13
    ir = L.bf16x_gesv_ir
    assert ir(4, None, 3, None, None, 3, 0, 0.0, 0, None, ctypes.byref(rep)) == -3
    assert ir(4, None, 4, None, None, 3, 0, float("nan"), 0, None, ctypes.byref(rep)) == -8
    assert ir(4, None, 4, None, None, 3, 0, 0.0, 0, None, None) == -11
    info = ctypes.c_int(0)
    f = L.bf16x_getrf
    assert f(-1, None, 1, None, 3, 0, ctypes.byref(info)) == -1
    assert f(4, None, 4, None, 3, 0, ctypes.byref(info)) == -2
    assert f(4, 16, 3, None, 3, 0, ctypes.byref(info)) == -3
    assert f(4, 16, 4, None, 3, 0, ctypes.byref(info)) == -4
    assert f(4, 16, 4, 32, 4, 0, ctypes.byref(info)) == -5
    import torch
    if not torch.cuda.is_available():
        assert f(4, 16, 4, 32, 3, 0, ctypes.byref(info)) == bx.ERR_ARCH
        assert g(4, 16, 4, 32, 48, 3, 0, 0, 0.0, 0.0, 0, None, ctypes.byref(rep)) == bx.ERR_ARCH

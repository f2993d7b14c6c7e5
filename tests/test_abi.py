"""C ABI: the library loads without a GPU, exports every symbol the header
declares, and its natively computed 1-D tables match the reference's."""

import os
import re

import numpy as np
import pytest

from helpers import load

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "wavekernel_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wk_[a-z_A-Z0-9]+)\s*\(", src)))


def test_library_exports_header_symbols():
    from paper_1805_03981_b200 import _lib
    lib = _lib.lib()
    names = _header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(_lib._SIGS), set(names) - set(_lib._SIGS)
    assert lib.wk_version() >= 1


def test_native_tables_match_reference():
    from paper_1805_03981_b200._lib import basis_table
    z = load("tables")
    for k in range(1, 13):
        s = k * k
        assert np.abs(basis_table("gauss_points", k) - z[f"gauss_points_{k}"]).max() < 1e-15
        assert np.abs(basis_table("gauss_weights", k) - z[f"gauss_weights_{k}"]).max() < 1e-15
        assert np.abs(basis_table("gl_points", k) - z[f"gl_points_{k}"]).max() < 1e-15
        assert np.abs(basis_table("gl_weights", k) - z[f"gl_weights_{k}"]).max() < 1e-15
        assert np.abs(basis_table("gl_to_g", k) - z[f"gl_to_g_{k}"]).max() < 1e-13
        assert np.abs(basis_table("g_to_gl", k) - z[f"g_to_gl_{k}"]).max() < 1e-13 * s
        assert np.abs(basis_table("d_gl", k) - z[f"d_gl_{k}"]).max() < 1e-13 * s
        assert np.abs(basis_table("d_co", k) - z[f"d_co_{k}"]).max() < 1e-13 * s
        for j in range(k + 1):
            assert np.abs(basis_table("resize", k, j) - z[f"proj_{k}_{j}"]).max() < 1e-13


def test_split_operator_identity():
    """A = 1/2 M1^{-1}(B^T W Dgl - Dgl^T W B) and the lift vectors, rebuilt
    from the reference tables (the collapsed affine cell operator)."""
    from paper_1805_03981_b200._lib import basis_table
    z = load("tables")
    for k in range(1, 9):
        B, Dg, w = z[f"gl_to_g_{k}"], z[f"d_gl_{k}"], z[f"gauss_weights_{k}"]
        M1 = B.T @ (w[:, None] * B)
        A = 0.5 * np.linalg.solve(M1, B.T @ (w[:, None] * Dg) - Dg.T @ (w[:, None] * B))
        assert np.abs(basis_table("a_split", k) - A).max() < 1e-11 * (k + 1) ** 2
        L = np.linalg.inv(M1)
        lift = basis_table("lift", k)
        assert np.abs(lift[0] - L[:, 0]).max() < 1e-11 * (k + 1) ** 2
        assert np.abs(lift[1] - L[:, -1]).max() < 1e-11 * (k + 1) ** 2


def test_operator_requires_cuda_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1805_03981_b200 as W
    mesh = W.build_cartesian(2, 2, "periodic")
    with pytest.raises(RuntimeError):
        W.AcousticOperator(mesh, W.affine_geometry(mesh, 2), W.Material.uniform(mesh),
                           device="cpu")

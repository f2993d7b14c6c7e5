"""Host-side 1-D rules (paper_1805_03981_b200/rules.py): the numpy long-double
Gauss / Gauss-Lobatto points used to BUILD problems are bit-identical to the
native tables the kernels use, and agree with the reference's tables
(tests/golden/tables.npz) to round-off; long-double Lagrange rows sum to
zero far below double round-off."""

import numpy as np
import pytest

from helpers import load
from paper_1805_03981_b200 import rules
from paper_1805_03981_b200._lib import basis_table


@pytest.mark.parametrize("k", range(1, 13))
def test_rules_bitwise_native_and_reference(k):
    assert np.array_equal(rules.gl_points(k), basis_table("gl_points", k))
    assert np.array_equal(rules.gauss_points(k), basis_table("gauss_points", k))
    assert np.abs(rules.gauss_weights(k) - basis_table("gauss_weights", k)).max() <= 2e-16
    z = load("tables")
    assert np.abs(rules.gl_points(k) - z[f"gl_points_{k}"]).max() < 1e-15
    assert np.abs(rules.gauss_points(k) - z[f"gauss_points_{k}"]).max() < 1e-15
    assert np.abs(rules.gauss_weights(k) - z[f"gauss_weights_{k}"]).max() < 1e-15


@pytest.mark.parametrize("g", [1, 3, 5, 8])
def test_lagrange_rows_long_double(g):
    nodes = np.array([0.0, 1.0]) if g == 1 else rules.gl_points(g)
    pts = rules.gauss_points(6)
    d = rules.lagrange_ld(nodes, pts, derivative=True)
    v = rules.lagrange_ld(nodes, pts)
    assert d.dtype == np.longdouble
    assert np.abs(d.sum(axis=1)).max() < 1e-16          # derivative of a constant
    assert np.abs(v.sum(axis=1) - 1).max() < 1e-17      # partition of unity

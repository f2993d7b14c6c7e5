"""Memory / index checking of the kernels (SURVEY.md §5 "race detection";
compute-sanitizer is not available on the GPU pool).

``libwk_b200_check.so`` is the same library built with -DWK_CHECK: every
neighbour / ghost index a kernel gathers through, the element range of every
tile (including the structured traversal) and the dynamic shared memory each
kernel's layout needs are asserted on the device, and a violation traps the
launch.  This test re-runs the parity suites (operators on every golden case,
steppers, curved geometry, general affine meshes with several tiles per CTA,
multi-slab ghost exchange, long trajectories) against that library in a
subprocess and requires them all to pass -- and the checked library to be the
one mapped."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_1805_03981_b200", "libwk_b200_check.so")

DRIVER = r"""
import os, sys
import pytest
sys.path.insert(0, {root!r})
from paper_1805_03981_b200 import _lib
_lib.lib()
maps = open("/proc/self/maps").read()
assert "libwk_b200_check.so" in maps, "checked library not mapped"
sys.exit(pytest.main(["-q", "-x", "-p", "no:cacheprovider", "-m", "gpu", "-k",
                      "(parity or stepper or geometry or general_affine or slabs or long or degrees)"
                      " and not checked",
                      os.path.join({root!r}, "tests")]))
"""


def test_parity_suites_under_checked_build(cuda):
    if not os.path.exists(CHECK_LIB):
        pytest.fail("libwk_b200_check.so missing: run __graft_entry__.build()")
    env = dict(os.environ, WK_LIB_PATH=CHECK_LIB)
    p = subprocess.run([sys.executable, "-c", DRIVER.format(root=ROOT)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1800)
    tail = (p.stdout + p.stderr)[-3000:]
    assert p.returncode == 0, tail
    assert "WK_CHECK failed" not in p.stdout + p.stderr, tail


NEGATIVE = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_1805_03981_b200 as W
from paper_1805_03981_b200 import _lib, configs
prob = configs.config("c2", scale=0.25)
op = W.AcousticOperator(prob.mesh, prob.geometry, prob.material)
_lib.check(_lib.lib().wk_debug_set_neighbor(op._ctx, 7, 1, prob.mesh.n_elements + 1000))
u = torch.from_numpy(prob.state).cuda()
op.rhs(W.StateVector(u, prob.k, 3))
torch.cuda.synchronize()
print("NO TRAP")
"""


def test_checked_build_traps_on_bad_neighbour(cuda):
    """A neighbour code past the mesh (planted behind the host validation)
    must trap the checked kernel; the production library has no device check."""
    env = dict(os.environ, WK_LIB_PATH=CHECK_LIB)
    p = subprocess.run([sys.executable, "-c", NEGATIVE.format(root=ROOT)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    out = p.stdout + p.stderr
    assert p.returncode != 0 and "NO TRAP" not in out, out[-2000:]
    assert "WK_CHECK failed" in out, out[-2000:]


def test_host_rejects_bad_neighbour_table(cuda):
    import numpy as np
    import paper_1805_03981_b200 as W
    from paper_1805_03981_b200 import configs, mesh as M
    prob = configs.config("c2", scale=0.125)
    bad = np.array(prob.mesh.neighbors)
    bad[3, 0, 1] = prob.mesh.n_elements
    m = M.Mesh(prob.mesh.d, prob.mesh.n_per_dim, prob.mesh.vertices, prob.mesh.elements, bad,
               prob.mesh.boundary_kind)
    with pytest.raises(ValueError, match="neighbour table"):
        W.AcousticOperator(m, prob.geometry, prob.material)

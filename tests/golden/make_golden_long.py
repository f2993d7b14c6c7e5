"""Long-trajectory golden fixtures: 100 time steps of the UNMODIFIED reference.

north_star's second parity bar is "1e-10 after 100 time steps".  This script
runs the reference's own stepper (``wavekernel.stepping.make_stepper`` /
``advance``, stepping.py:288-308) for 100 steps on

* 8^3 versions of the config 2, 3 and 4 rules and a 16x16x8 version of the
  config 5 rules (both schemes where the config names two), and
* config 2 at its FULL BASELINE size (32^3, k=4, 16.4 M DoF; ~1 h of CPU),

with the same frozen inputs the GPU path uses (``paper_1805_03981_b200.
configs``).  Config 3 feeds the reference's unchanged ``AcousticOperator`` a
geometry from ``oracle.precompute_geometry`` (the reference mesh code cannot
build the degree-5 map).

To keep the fixtures small, each stores the final state at 128 (full c2: 256)
seeded sampled elements, plus full-state checksums: the per-component sum of
squares and the mass-matrix norm of the final state (``state_norm``,
stepping.py:321-324).  Run in the build container:

    python tests/golden/make_golden_long.py [case ...]
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from wavekernel import mesh as RM, operator as RO, stepping as RS  # noqa: E402
from wavekernel.operator import StateVector  # noqa: E402

from make_golden import _oracle_geometry  # noqa: E402
from paper_1805_03981_b200 import configs  # noqa: E402

LONG = [
    # name, config, scale, scheme, steps, sampled elements
    ("c2s8_lsrk45_100", "c2", 0.25, "lsrk45", 100, 128),
    ("c3s8_ader_hdg_100", "c3", 0.25, "ader_hdg", 100, 128),
    ("c4s8_ader_hdg_100", "c4", 1 / 6, "ader_hdg", 100, 128),
    ("c4s8_lsrk45_100", "c4", 1 / 6, "lsrk45", 100, 128),
    ("c5s16_lsrk45_100", "c5", 0.125, "lsrk45", 100, 128),
    ("c5s16_ader_hdg_100", "c5", 0.125, "ader_hdg", 100, 128),
    ("c2full_lsrk45_100", "c2", 1.0, "lsrk45", 100, 256),
]


def sample_ids(n_elements: int, count: int) -> np.ndarray:
    """First, last and seeded random elements (shared with the GPU test)."""
    rng = np.random.default_rng(20261020)
    ids = {0, n_elements - 1}
    while len(ids) < min(count, n_elements):
        ids.add(int(rng.integers(0, n_elements)))
    return np.asarray(sorted(ids), dtype=np.int64)


def run(name, cfg, scale, scheme, steps, count):
    t0 = time.time()
    prob = configs.config(cfg, scale=scale)
    m = prob.mesh
    rmesh = RM.Mesh(m.d, m.n_per_dim, m.vertices, m.elements, m.neighbors, [],
                    m.boundary_kind)
    k = prob.k
    reduced = RS.reduction_degrees(k, "every_second")
    if cfg == "c3":
        base = RM.build_cartesian(m.n_per_dim, 3, "periodic")
        geo = _oracle_geometry(base, k, 5, configs.c3_mapping, reduced)
    else:
        geo = RM.precompute_geometry(rmesh, k, reduced_degrees=reduced)
    mat = RM.Material(c=prob.material.c, rho=prob.material.rho)
    op = RO.AcousticOperator(rmesh, geo, mat)
    cr = prob.schemes[scheme][0]
    dt = RS.compute_dt(cr, rmesh, mat, k)
    stepper = RS.make_stepper(RS.SchemeConfig(scheme=scheme, courant=cr), op)
    st = StateVector(prob.state.copy(), k, m.d)
    t1 = time.time()
    st = RS.advance(st, dt, steps, stepper)
    t2 = time.time()
    u = st.data
    ids = sample_ids(m.n_elements, count)
    np.savez_compressed(
        os.path.join(HERE, f"long_{name}.npz"), config=cfg, scale=scale, scheme=scheme,
        steps=steps, dt=dt, courant=cr, n_elements=m.n_elements, ids=ids,
        u0_sumsq=np.sum(prob.state ** 2), u_sample=u[ids],
        sumsq=np.sum(u ** 2, axis=tuple(i for i in range(u.ndim) if i != 1)),
        norm=RS.state_norm(op, st), setup_s=t1 - t0, run_s=t2 - t1)
    print(f"{name}: {m.n_elements} elements, setup {t1 - t0:.1f} s, "
          f"{steps} steps {t2 - t1:.1f} s", flush=True)


if __name__ == "__main__":
    only = set(sys.argv[1:])
    for case in LONG:
        if not only or case[0] in only:
            run(*case)

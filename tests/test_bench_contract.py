"""bench.py contract checks that need no GPU: the CPU reference arm builds its
inputs and runs the oracle without loading the product library, and both arms
describe the workload with the same ``config`` object."""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_does_not_load_product_library():
    code = ("import bench\n"
            "prob, om, op = bench._oracle_problem('c5', 1 / 16)\n"
            "op.rhs(prob.state)\n"
            "print('LOADED' if 'libwk_b200' in open('/proc/self/maps').read() else 'CLEAN')\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "CLEAN"


def test_workload_config_is_shared():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.workload_config("c5", "lsrk45", 1)
    assert a == bench.workload_config("c5", "lsrk45", 1)
    assert a["dofs"] == 128 * 128 * 64 * 4 * 125
    assert bench.workload_config("c5", "lsrk45", 8)["parallelism"].startswith("8 x-slabs")
    assert bench.DEFAULT_SCHEME["c5"] == "lsrk45"

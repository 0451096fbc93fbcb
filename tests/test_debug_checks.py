"""Bounds and single-writer checks of the scatter paths (SURVEY §5 race /
memory checking; compute-sanitizer is closed on this GPU pool): the library
built with EPFEM_DEBUG_CHECKS=1 (device asserts: every row-stream add lands
inside the segment of the node its warp owns, record blocks inside their
element record, range sizes within the plan) runs the parity tests of every
element type and BASELINE configuration in a fresh interpreter; a failed
device assert aborts the kernel, so the subprocess must pass."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parity_suite_under_debug_checks(cuda):
    from paper_1805_04155_b200 import build as B
    lib = B.build(debug_checks=True)
    env = dict(os.environ, EPFEM_GPU_LIB=lib)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-k", "pattern_and_elastic or tangent_matches or fused_step_all or config_pipeline or "
                              "slab_ranks or single_cell or strains_and_internal"],
                       env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout

"""Sanitizer-substitute tier (compute-sanitizer is closed on the GPU pool): every kernel family
(tools/sanitize_case.py) through the checked library libspaimg_cuda_debug.so, which starts all
level buffers and the coarse engines' shared arrays with NaN interiors and slack (zero frames
only) and puts random per-warp delays at every mbarrier wait and engine barrier.  A read before
write, a read outside the stencil's reach, or a missing barrier turns into a NaN or a
nondeterministic value, and the case's bitwise comparisons with the C oracle fail.  Run twice
with the marching kernels forced on every level and twice with the default flat kernels."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", ["march", "flat"])
@pytest.mark.parametrize("rep", [0, 1])
def test_checked_build_bitwise(mode, rep):
    env = dict(os.environ, SPAIMG_DEBUG="1")
    if mode == "march":
        # ... and the K3 + K1 marches (in-place correction of the staged rows / planes) on every level
        env.update(SPAIMG_FLAT_N2="0", SPAIMG_FLAT_N3="0", SPAIMG_PC2_N="1", SPAIMG_PC3_N="1")
    code = ("import runpy, sys; sys.argv = ['sanitize_case']; "
            "from paper_2206_05543_b200 import _lib; lib = _lib.load(); "
            "assert _lib.LIB_PATH.endswith('libspaimg_cuda_debug.so'), _lib.LIB_PATH; "
            "runpy.run_path('tools/sanitize_case.py', run_name='__main__')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, env=env,
                       timeout=900)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "ok all" in r.stdout

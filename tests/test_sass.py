"""SASS guard of the bitwise contract: no fused multiply-add
in any kernel that computes the iterate or the coarse right-hand side.  FMAs are allowed only
where they are part of the contract or off the iterate path:
  * the coarse LU solve (getrs order with FMA, Appendix A.6, and the correctly rounded pivot
    division): k_coarse_solve, k_tail, k_tail_fast;
  * the residual norm's sqrt (IEEE-rounded sqrt uses DFMA internally; the norm never feeds back):
    the Mode 1/2 (norm) instantiations of the marching kernels, the NORM variants of the flat
    tile sweeps, k_residual_norm.
Runs on the CPU with cuobjdump on the in-tree library."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2206_05543_b200", "libspaimg_cuda.so")


def _fma_counts():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool) or not os.path.exists(LIB):
        pytest.skip("cuobjdump or the built library is missing")
    sass = subprocess.run([tool, "-sass", LIB], capture_output=True, text=True, check=True).stdout
    counts, fn = {}, None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            fn = m.group(1)
            counts.setdefault(fn, 0)
        elif fn and re.search(r"\b[DF]FMA\b", line):
            counts[fn] += 1
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.split("\n")
    return {n: counts[m] for n, m in zip(names, counts)}


def _allowed(name):
    if any(k in name for k in ("k_coarse_solve", "k_tail<", "k_tail_fast<", "k_residual_norm")):
        return True
    m = re.match(r"void spaimg::k_sweep(2d|3d)_march<\w+, \d+, (true|false), (\d)(, (true|false))?>", name)
    if m:
        return m.group(3) in ("1", "2")  # norm modes
    m = re.match(r"void spaimg::k_sweep(2d|3d)_tile<\w+, \d+, (true|false), (true|false)>", name)
    if m:
        return m.group(3) == "true"  # the flat sweep's norm variant (NORM = true)
    return False


def test_no_fma_on_the_iterate_path():
    counts = _fma_counts()
    assert len(counts) > 50
    bad = {n: c for n, c in counts.items() if c and not _allowed(n)}
    assert not bad, bad
    # the guard sees the kernels it is meant to guard
    hot = [n for n in counts if any(k in n for k in ("k_sweep2d_march", "k_sweep3d_march", "k_residual_restrict2d",
                                                      "k_prolong_correct2d", "k_rr2d_flat", "k_sweep2d_tile"))]
    assert len(hot) > 20
    # and the getrs-order LU does use FMA, as OpenBLAS does (Appendix A.6)
    assert all(c > 0 for n, c in counts.items() if "k_coarse_solve" in n)

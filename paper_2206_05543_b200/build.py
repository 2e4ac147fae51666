"""In-tree build of libspaimg_cuda.so (sm_100a) with nvcc.

    python -m paper_2206_05543_b200.build [--force] [--debug]

The library has a plain C ABI (include/spaimg_cuda.h), links the CUDA runtime
statically (so it does not depend on torch's libcudart), and is loaded with ctypes.
"""

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libspaimg_cuda.so")
# checked build (-DSPAIMG_DEBUG_CHECKS; NaN poisoning + barrier jitter, spaimg_common.cuh),
# loaded instead of LIB when SPAIMG_DEBUG=1
LIB_DEBUG = os.path.join(PKG, "libspaimg_cuda_debug.so")

SOURCES = ["kernels_basic.cu", "kernels_sweep.cu", "kernels_sweep_pc.cu", "kernels_sweep2.cu", "kernels_sweep3d.cu", "kernels_restrict.cu", "kernels_tail.cu", "kernels_tail_fast2d.cu", "kernels_tail_fast3d.cu", "kernels_flat.cu", "kernels_rng.cu", "solver.cu"]
HEADERS = ["spaimg_common.cuh", "kernels.h", "ptx.cuh", "march.cuh", "sweep2d_march.cuh", "tail_ops.cuh", "kernels_tail_fast.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "--fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
]


def nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(INCLUDE, "spaimg_cuda.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps)


def _obj_stale(src, obj):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    deps += [os.path.join(INCLUDE, "spaimg_cuda.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, obj, debug=False):
    flags = ["-DSPAIMG_DEBUG_CHECKS"] if debug else []
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *flags, "-I", INCLUDE, "-I", CSRC, "-c", os.path.join(CSRC, src), "-o", obj]
    return src, subprocess.run(cmd, capture_output=True, text=True)


def build(force=False, verbose=False, debug=False):
    """Compile the stale objects in parallel (one nvcc per source), then link.  debug=True
    builds the checked library (LIB_DEBUG) from its own objects."""
    lib = LIB_DEBUG if debug else LIB
    if not force and not _stale(lib):
        return lib
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build", "debug") if debug else os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, src.replace(".cu", ".o")) for src in SOURCES]
    todo = [(s, o) for s, o in zip(SOURCES, objs) if force or _obj_stale(s, o)]
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for src, r in ex.map(lambda so: _compile(*so, debug=debug), todo):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
    tmp = lib + ".tmp"
    cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))

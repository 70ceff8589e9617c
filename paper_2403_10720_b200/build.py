"""Build libdvc.so in-tree for sm_100a (explicit nvcc; no JIT cache, so the
built library travels to the GPU box with the repo snapshot).

    python -m paper_2403_10720_b200.build [--verbose]
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdvc.so")
SOURCES = ["api.cu", "kernels.cu", "host.cpp", "mcts.cpp"]
HEADERS = ["dvc_internal.h", "rollout.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c


def _stale(lib=LIB):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "dvc.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


LIB_DEBUG = os.path.join(HERE, "libdvc_debug.so")


def build(force=False, verbose=False, debug=False):
    """Release libdvc.so, or (debug=True) libdvc_debug.so with the device-side
    invariant checks (-DDVC_DEBUG; dvc_debug_counters)."""
    out = LIB_DEBUG if debug else LIB
    if not force and not _stale(out):
        return out
    tmp = out + ".tmp.%d" % os.getpid()
    cmd = [_nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-O2", "-Xcompiler", "-ffp-contract=off", "-I", os.path.join(HERE, "..", "include"), "-o", tmp]
    if debug:
        cmd += ["-DDVC_DEBUG"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += [os.path.join(CSRC, f) for f in SOURCES]
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv, debug="--debug" in sys.argv))

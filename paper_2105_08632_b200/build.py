"""Build libsdrt.so in-tree with nvcc for sm_100a (no torch extension machinery)."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
PROF = os.environ.get("SDRT_PHASE_PROF") == "1"  # tools-only phase-cycle build
# tools-only tuning variants: SDRT_VARIANT=name SDRT_DEFS="-DFOO=1" -> libsdrt_<name>.so
VARIANT = os.environ.get("SDRT_VARIANT", "prof" if PROF else "")
EXTRA_DEFS = os.environ.get("SDRT_DEFS", "").split()
OUT = os.path.join(HERE, f"libsdrt_{VARIANT}.so" if VARIANT else "libsdrt.so")
BUILD = os.path.join(HERE, f"build_{VARIANT}" if VARIANT else "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v"] + (["-DSDRT_PHASE_PROF"] if PROF else []) + EXTRA_DEFS
CXX_FLAGS = ["-O2", "-std=gnu++17", "-fPIC", "-Wall"]
INCLUDES = ["-I" + os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "include")]
LINK_LIBS = ["-lquadmath", "-lcudart", "-ldl"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _nvcc():
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def _stamp():
    """Flags + defines the library is built with; a change forces a rebuild."""
    return hashlib.sha1(" ".join(ARCH + NVCC_FLAGS + CXX_FLAGS + LINK_LIBS).encode()).hexdigest()


def _compile(s):
    o = os.path.join(BUILD, os.path.basename(s) + ".o")
    if s.endswith(".cu"):
        cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *INCLUDES, "-c", s, "-o", o]
    else:
        cmd = ["g++", *CXX_FLAGS, *INCLUDES, "-c", s, "-o", o]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return o, r.returncode, " ".join(cmd) + "\n" + r.stdout + r.stderr


def build(verbose=False, force=False):
    srcs = sources()
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(HERE, "..", "include", "sdrt.h"))
    stamp_file = OUT + ".stamp"
    if not force and os.path.exists(OUT) and os.path.exists(stamp_file):
        t = os.path.getmtime(OUT)
        if open(stamp_file).read() == _stamp() and all(os.path.getmtime(f) < t for f in srcs + hdrs):
            return OUT
    os.makedirs(BUILD, exist_ok=True)
    # largest translation units first so the pool stays busy
    order = sorted(srcs, key=lambda f: -os.path.getsize(f))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = dict(zip(order, ex.map(_compile, order)))
    objs, logs = [], []
    for s in srcs:
        o, rc, log = results[s]
        logs.append(log)
        if rc != 0:
            sys.stderr.write(log)
            raise RuntimeError(f"compile failed: {s}")
        objs.append(o)
    cmd = [_nvcc(), *ARCH, "-shared", "-o", OUT, *objs, *LINK_LIBS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    logs.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(logs[-1])
        raise RuntimeError("link failed")
    with open(stamp_file, "w") as f:
        f.write(_stamp())
    with open(os.path.join(BUILD, "build.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force=True)
    print(OUT)

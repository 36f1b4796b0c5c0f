"""Build libpwb200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Usage:  python -m paper_2505_02319_b200.build [--force] [--variant NAME -DMACRO=VALUE ...]

A variant (performance experiments only) is built into libpwb200_<NAME>.so and
selected at load time with PWB200_VARIANT=<NAME>; the default library is the
product.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpwb200.so")
SOURCES = ["grid.cu", "fft_kernels.cu", "proj.cu", "state.cu", "cg.cu", "chi0.cu", "vec.cu", "comm.cu", "projw.cu"]
HEADERS = ["common.cuh", "fft_engine.cuh", "grid.cuh", "proj.cuh", "state.cuh", "profile.cuh", "fft_static.cuh", "dispatch.cuh", "tma.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "--expt-relaxed-constexpr"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def lib_path(variant=""):
    return os.path.join(HERE, f"libpwb200_{variant}.so" if variant else "libpwb200.so")


def _stale(lib):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "pwb200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, variant="", defines=()):
    """Compile every CUDA source for sm_100a and link libpwb200.so next to this file."""
    lib = lib_path(variant)
    if not force and not _stale(lib):
        return lib
    nvcc = _nvcc()
    objdir = os.path.join(HERE, "build" + (f"_{variant}" if variant else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc, *NVCC_FLAGS, *defines, "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{out.decode()}")
        if verbose and out:
            print(out.decode())
    tmp = lib + ".tmp"
    cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs,
           "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    argv = sys.argv[1:]
    var = argv[argv.index("--variant") + 1] if "--variant" in argv else ""
    defs = tuple(a for a in argv if a.startswith("-D"))
    print(build(force="--force" in argv or bool(var), verbose="-v" in argv, variant=var,
                defines=defs))

"""Build libmpcb200.so in-tree with nvcc for sm_100a.

    python -m paper_2403_16013_b200.build [--verbose-ptxas]

Each translation unit (the per-K kernel instantiations and the C-ABI) is
compiled in parallel; the shared object lands in
paper_2403_16013_b200/lib/libmpcb200.so (git-ignored, travels to the GPU
box with the gpurun snapshot).  --fmad=false is a belt-and-braces guard: the
kernels already use explicit round-to-nearest intrinsics, so the only DFMA in
the SASS is TwoProd's error term.
"""

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
OBJDIR = os.path.join(HERE, "lib", "obj")
LIB = os.path.join(LIBDIR, "libmpcb200.so")

SOURCES = ["inst_k2.cu", "inst_k3.cu", "inst_k4.cu", "inst_k5.cu", "inst_k6.cu", "inst_k8.cu", "abi.cu", "ozaki.cu", "ozaki_tc.cu", "mgpu.cu", "metrics.cu"]
HEADERS = ["expansion.cuh", "kernels.cuh", "ops.h", "prof.h", "sortnet.h", "abi_util.h", "inst_hik.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-O2", "--expt-relaxed-constexpr"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS]
    if src in ("ozaki.cu", "ozaki_tc.cu"):
        deps.append(os.path.join(CSRC, "ozaki_tc.h"))
    if src in ("abi.cu", "ozaki.cu", "mgpu.cu", "metrics.cu"):
        deps.append(os.path.join(os.path.dirname(HERE), "include", "mpc_b200.h"))
    if not _stale(obj, deps):
        return obj, ""
    cmd = [nvcc()] + ARCH + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + [
        "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose=False, force=False):
    os.makedirs(OBJDIR, exist_ok=True)
    if force:
        for f in os.listdir(OBJDIR):
            os.remove(os.path.join(OBJDIR, f))
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    objs = [o for o, _ in results]
    logs = "".join(l for _, l in results)
    if _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-lcudart_static", "-lcublas", "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-lrt",
            "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB, logs


if __name__ == "__main__":
    lib, logs = build(verbose="--verbose-ptxas" in sys.argv, force="--force" in sys.argv)
    if logs:
        print(logs)
    print(lib)

"""Build libsv.so (hand-written CUDA for sm_100a + NCCL) in-tree with nvcc.

python paper_quant_ph_9804039_b200/build.py [--force] [--verbose] [-DMACRO=V --out=PATH]
Compiles every csrc/*.cu and csrc/*.cpp to an object (in parallel) and links
paper_quant_ph_9804039_b200/libsv.so; objects and the .so are git-ignored but
travel to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libsv.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl  # the NCCL 2.28 wheel torch uses

    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    raise RuntimeError("nvcc not found")


def _compile(src: str, verbose: bool, objdir: str = OBJ, defines=()) -> str:
    inc, _ = _nccl_dirs()
    obj = os.path.join(objdir, os.path.basename(src) + ".o")
    deps = [src] + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "sv.h")
    ]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
           "-I", inc, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    if src.endswith(".cu"):
        cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
    else:
        cmd += ["-x", "c++"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """defines/out: an alternative build (e.g. SV_TILE_MIN_BLOCKS=3) into its
    own object directory and .so, loadable with SV_LIB=<path> for A/B runs."""
    lib = out or LIB
    objdir = OBJ if not defines else os.path.join(OBJ, "_".join(d.replace("=", "") for d in defines))
    os.makedirs(objdir, exist_ok=True)
    if force:
        for f in glob.glob(os.path.join(objdir, "*.o")):
            os.remove(f)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, objdir, defines), srcs))
    _, libdir = _nccl_dirs()
    if force or not os.path.exists(lib) or os.path.getmtime(lib) < max(os.path.getmtime(o) for o in objs):
        cuda_lib = os.path.join(os.path.dirname(os.path.dirname(_nvcc())), "lib64")
        cmd = [_nvcc(), *ARCH, "-shared", "-o", lib, *objs, "-L", libdir, "-l:libnccl.so.2",
               "-lnvrtc", "-ldl", "-Xlinker", f"-rpath,{libdir}", "-Xlinker", f"-rpath,{cuda_lib}"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
                out=outs[0] if outs else None))

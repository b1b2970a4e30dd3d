"""Build libzf.so (the product library) and synth/libzfsynth.so (input generator) in-tree.

nvcc cross-compiles for sm_100a without a GPU.  The built .so files are
git-ignored but travel to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIBZF = os.path.join(PKG, "libzf.so")
LIBSYNTH = os.path.join(ROOT, "synth", "libzfsynth.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    raise RuntimeError("NCCL (nvidia.nccl wheel) not found")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl = _nccl_dir()
    extra = os.environ.get("ZF_NVCC_EXTRA", "").split()
    common = ARCH + extra + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-ffp-contract=off,-fno-math-errno", "-Xptxas", "-v" if verbose else "-O3",
                     "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include")]
    # a change of compile flags (e.g. ZF_NVCC_EXTRA experiments) forces a rebuild
    stamp = os.path.join(BUILD, "flags.txt")
    flags = " ".join(common).replace(ROOT, "<root>")   # a copy of the tree reuses its objects
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + [os.path.join(ROOT, "include", "zf.h")]
    objs = []
    jobs = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC] + common + ["-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return r

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(LIBZF, objs):
        run([NVCC] + ARCH + ["-shared", "-o", LIBZF + ".tmp"] + objs +
            ["-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", "-Xlinker", f"-rpath,{os.path.join(nccl, 'lib')}",
             "-lpthread"])
        os.replace(LIBZF + ".tmp", LIBZF)
    with open(stamp, "w") as f:
        f.write(flags)
    synth_src = os.path.join(ROOT, "synth", "synth.cu")
    if force or _stale(LIBSYNTH, [synth_src]):
        run([NVCC] + ARCH + ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", synth_src, "-o", LIBSYNTH + ".tmp"])
        os.replace(LIBSYNTH + ".tmp", LIBSYNTH)
    return LIBZF


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIBZF)

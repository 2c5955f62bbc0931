"""In-tree build of libdsel.so (sm_100a) -- called by __graft_entry__.build().

nvcc compiles the CUDA engine for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo; the host RNG is compiled by g++ with -ffp-contract=off (it
must reproduce the reference's Box-Muller bits). NCCL is the torch-bundled
2.28 (same library torch.distributed loads), linked with an rpath.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "lib")
LIB = os.path.join(OUT, "libdsel.so")
CLI = os.path.join(OUT, "doptsel")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]


def up_to_date(target, deps):
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    inc = os.path.join(ROOT, "include")
    nccl_inc, nccl_lib = nccl_dirs()
    deps = sources() + [os.path.join(inc, "dsel.h"), __file__,
                        os.path.join(PKG, "tools", "doptsel_main.cpp")]
    if not force and up_to_date(LIB, deps):
        return LIB
    objs = []
    nv = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
          "-I", inc, "-I", nccl_inc, "--expt-relaxed-constexpr"]
    if verbose_ptxas:
        nv += ["-Xptxas", "-v"]
    o = os.path.join(OUT, "engine.o")
    _run(nv + ["-c", os.path.join(CSRC, "engine.cu"), "-o", o])
    objs.append(o)
    for cpp in ("host_rng.cpp", "lti.cpp", "kbf.cpp"):
        src = os.path.join(CSRC, cpp)
        if not os.path.exists(src):
            continue
        o = os.path.join(OUT, cpp.replace(".cpp", ".o"))
        _run(["g++", "-O3", "-std=gnu++20", "-fPIC", "-ffp-contract=off", "-pthread", "-I", inc,
              "-c", src, "-o", o])
        objs.append(o)
    _run(["nvcc", *ARCH, "-shared", "-o", LIB, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
          "-Xlinker", "-rpath=" + nccl_lib, "-Xcompiler", "-pthread"])
    for o in objs:
        os.remove(o)
    build_cli()
    return LIB


def build_cli() -> str:
    """The drop-in `doptsel select` CLI (tools/doptsel_main.cpp) over libdsel.so."""
    src = os.path.join(PKG, "tools", "doptsel_main.cpp")
    _run(["g++", "-O2", "-std=gnu++20", "-Wall", "-I", os.path.join(ROOT, "include"), src,
          "-o", CLI, "-L", OUT, "-ldsel", "-Wl,-rpath,$ORIGIN", "-pthread"])
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)

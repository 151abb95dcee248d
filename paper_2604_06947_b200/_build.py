"""Build libfqnm.so (the C-ABI library) in-tree with nvcc for sm_100a.

Every translation unit is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
and the Euler/Roe kernels additionally with -fmad=false (pinned binary64
operation order, reading R-ROE).  cudart is linked statically.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfqnm.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-diag-suppress", "177", "-Xcompiler", "-fPIC", "-I", CSRC, "-I", INCLUDE]
# (object name, source, extra flags)
UNITS = {
    "fqnm_api.cu": [],
    # kernels_scalar.cu is compiled as 10 parts (separate objects, -DFQNM_SCALAR_PART=k) in
    # parallel: each part holds a subset of the launchers' template instantiations
    **{f"kernels_scalar_p{k}.cu": [f"-DFQNM_SCALAR_PART={k}"] for k in range(1, 11)},
    "kernels_euler.cu": ["-fmad=false"],
    "kernels_diag.cu": [],
    "kernels_3d.cu": [],
    "kernels_3d_s.cu": [],
    "kernels_2d.cu": [],
}
HEADERS = ["fqnm_internal.h", "maps.cuh", "kernels_scalar.cu"]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "fqnm.h"),
                                                               __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False,
          defines=(), lib: str = LIB, objdir: str = "") -> str:
    objdir = objdir or os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    cmds = []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, "kernels_scalar.cu" if unit.startswith("kernels_scalar_p") else unit)
        obj = os.path.join(objdir, unit.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, src):
            cmd = [NVCC, *ARCH, *COMMON, *extra, *[f"-D{x}" for x in defines], "-c", src, "-o", obj]
            if ptxas_v:
                cmd[1:1] = ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            cmds.append(cmd)
    rebuilt = bool(cmds)
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    if rebuilt or force or not os.path.exists(lib):
        tmp = lib + f".{os.getpid()}.tmp"
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"])
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, ptxas_v="-v" in sys.argv))

"""Build variants/libfqnm_<name>.so: recompile the named translation units with extra -D
defines and link them with the up-to-date objects of the main build (seconds, not minutes).
usage: python tools/build_variant.py <name> <unit.cu>[,<unit.cu>...] [DEFINE[=v] ...]
Select at run time with FQNM_LIBPATH=variants/libfqnm_<name>.so."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_06947_b200 import _build as B


def main():
    name, units, defines = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
    B.build()                                           # main objects up to date
    objdir = os.path.join(ROOT, "variants", "obj_" + name)
    os.makedirs(objdir, exist_ok=True)
    objs, cmds = [], []
    for unit, extra in B.UNITS.items():
        src = os.path.join(B.CSRC, "kernels_scalar.cu" if unit.startswith("kernels_scalar_p") else unit)
        base = "kernels_scalar.cu" if unit.startswith("kernels_scalar_p") else unit
        if base in units or unit in units:
            obj = os.path.join(objdir, unit.replace(".cu", ".o"))
            cmds.append([B.NVCC, *B.ARCH, *B.COMMON, *extra, *os.environ.get("NVCC_EXTRA", "").split(),
                         *[f"-D{d}" for d in defines], "-c", src, "-o", obj])
        else:
            obj = os.path.join(B.HERE, "build", unit.replace(".cu", ".o"))
        objs.append(obj)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        for f in [ex.submit(subprocess.check_call, c) for c in cmds]:
            f.result()
    lib = os.path.join(ROOT, "variants", f"libfqnm_{name}.so")
    subprocess.check_call([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-cudart", "static"])
    print(lib)


if __name__ == "__main__":
    main()

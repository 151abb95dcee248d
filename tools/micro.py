"""Build and run tools/micro.cu on the GPU, check the SASS of each kernel (one instruction
class per kernel), and write profiles/<tag>_micro.json: per-pipe issue rates in lane-ops
per SM clock (clock-independent; clock64 spans), with the SM clocks sampled during the
run.  bench.py reports its roofline against these measured rates as well as against the
theoretical issue peak (148 SMs x 128 lanes/clk).
usage: python tools/micro.py [tag]   (default tag r02)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EXPECT = {  # kernel symbol fragment -> SASS opcode that must dominate its loop
    "k_iadd3": "IADD3", "k_lop3": "LOP3.LUT", "k_imad": "IMAD", "k_imad_hi": "IMAD.HI",
    "k_ffma": "FFMA", "k_dfma": "DFMA", "k_i2fp": "I2FP.F32.S32", "k_lea_hi": "LEA.HI.SX32",
    "k_shfl": "SHFL.UP",
}


def build():
    exe = os.path.join(ROOT, "tools", "micro")
    src = os.path.join(ROOT, "tools", "micro.cu")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                               "-O3", "-std=c++17", "-I", os.path.join(ROOT, "paper_2604_06947_b200", "csrc"),
                               "-I", os.path.join(ROOT, "include"), src, "-o", exe])
    return exe


def sass_counts(exe):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", exe], capture_output=True,
                         text=True).stdout
    counts, cur = {}, None
    for line in out.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            counts[cur] = {}
            continue
        parts = line.split("*/")
        if cur and len(parts) > 1 and parts[0].strip().startswith("/*"):
            op = parts[1].strip().split(" ")[0].rstrip(";")
            if op and op[0].isalpha():
                counts[cur][op] = counts[cur].get(op, 0) + 1
    return counts


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    exe = build()
    sass = sass_counts(exe)
    checks = {}
    for frag, op in EXPECT.items():
        name = next((k for k in sass if frag + "P" in k), None)
        top = max(sass[name].items(), key=lambda kv: kv[1]) if name else None
        checks[frag] = {"expected": op, "top_op": top[0] if top else None,
                        "count": top[1] if top else 0}
    from bench import Clocks
    clk = Clocks(0)
    clk.start()
    res = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    c = clk.stop()
    rows = {}
    for line in res.splitlines():
        d = json.loads(line)
        rows[d.pop("name")] = d
    doc = {"what": "per-pipe issue rates on one B200: lane-ops per SM clock (clock64 spans of "
                   "co-resident CTAs, 32 warps/SM, 8 independent chains per thread)",
           "theoretical_issue_lane_ops_per_clk_per_sm": 128,
           "clocks": c, "sass_check": checks, **rows}
    path = os.path.join(ROOT, "profiles", f"{tag}_micro.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()

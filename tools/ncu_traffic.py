"""Extract per-launch DRAM traffic of a captured kernel from an ncu report into
profiles/<name>.json (read by bench.py for the roofline "traffic" field).
usage: python tools/ncu_traffic.py <report.ncu-rep> <out.json> [note]"""
import csv
import json
import subprocess
import sys


def main():
    rep, out = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}

    def num(key, scale):
        v, u = d[key]
        v = float(v.replace(",", ""))
        return v * scale.get(u, 1.0)

    byte_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    time_scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    res = {
        "kernel": d.get("Kernel Name", ("?", ""))[0],
        "grid": d.get("launch__grid_size", ("?", ""))[0],
        "registers": d.get("launch__registers_per_thread", ("?", ""))[0],
        "dram_bytes_read": num("dram__bytes_read.sum", byte_scale),
        "dram_bytes_write": num("dram__bytes_write.sum", byte_scale),
        "duration_ms": num("gpu__time_duration.sum", time_scale),
        "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]),
        "alu_pipe_pct": float(d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"][0]),
        "fma_pipe_pct": float(d["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"][0]),
        "source": rep.split("/")[-1], "note": note,
    }
    res["dram_bytes_per_launch"] = res["dram_bytes_read"] + res["dram_bytes_write"]
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

"""Write profiles/aty_fast_traffic.json from an `ncu --set full` capture of one
aty_fast_kernel launch (read by bench.py for roofline.traffic).

    python tools/traffic_json.py gpurun_out/prof_final.ncu-rep --n 100000 --p 1000000 \
        --format base-3
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
        "dram__bytes_read.sum.per_second", "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--n", type=int, required=True)
    ap.add_argument("--p", type=int, required=True)
    ap.add_argument("--format", default="2-bit", choices=["2-bit", "base-3"])
    ap.add_argument("--missing", type=float, default=0.0)
    ap.add_argument("--command", default="python bench.py --steps 1 --warmup 3 --no-cpu")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "aty_fast_traffic.json"))
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    metrics = {k: {"value": vals[head.index(k)], "unit": units[head.index(k)]}
               for k in KEEP if k in head}

    def nbytes(k):
        m = metrics[k]
        return float(m["value"].replace(",", "")) * SCALE[m["unit"]]
    nb = (a.n + 3) // 4
    xb = a.p * ((a.n + 4) // 5) if a.format == "base-3" else a.p * nb
    rec = {"kernel": "gi::aty_fast_kernel",
           "command": a.command + " (ncu --set full --clock-control none -k regex:aty_fast "
                      "-s 5 -c 1)",
           "n": a.n, "p": a.p, "format": a.format, "missing": a.missing,
           "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") +
           nbytes("dram__bytes_write.sum"),
           "algorithmic_bytes_per_launch": xb + 8 * a.n + 24 * a.p,
           "metrics": metrics}
    with open(a.out, "w") as fh:
        json.dump(rec, fh, indent=1)
        fh.write("\n")
    print(json.dumps({k: rec[k] for k in ("format", "dram_bytes_per_launch",
                                          "algorithmic_bytes_per_launch")}))


if __name__ == "__main__":
    main()

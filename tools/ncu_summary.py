"""Summarise an ncu capture of the sweep kernel into profiles/ncu_sweep_summary.json
(the `traffic` source of bench.py's roofline) and copy the launch list.

usage: python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv CONFIG ROUND [ALGO_BYTES]
"""
import csv
import io
import json
import os
import shutil
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, vals = rows[0], rows[2]
    return dict(zip(head, vals)), dict(zip(head, rows[1]))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(v) * scale


def main():
    rep, launches, cfg, rnd = sys.argv[1:5]
    algo = int(sys.argv[5]) if len(sys.argv) > 5 else None
    m, u = raw_metrics(rep)
    rd = to_bytes(m["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
    wr = to_bytes(m["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    dur = float(m["gpu__time_duration.sum"]) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}[u["gpu__time_duration.sum"]]
    times = []
    with open(launches) as f:
        for row in csv.DictReader(l for l in f if not l.startswith("==")):
            if row["Metric Name"] == "gpu__time_duration.sum" and "sweep_kernel" in row["Kernel Name"]:
                times.append(float(row["Metric Value"]) / 1e3)
    dst = os.path.join(ROOT, "profiles", f"launches_{rnd}_{cfg}.csv")
    shutil.copyfile(launches, dst)
    summ = {
        "kernel": m["Kernel Name"],
        "capture": "ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 3 -c 1",
        "command": "python bench.py --steps 5 --warmup 3 --no-solve --no-cpu-baseline",
        "duration_us": dur,
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "dram_bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": algo,
        "dram_throughput_pct_of_peak": float(m.get("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "nan")),
        "sm_throughput_pct": float(m["sm__throughput.avg.pct_of_peak_sustained_elapsed"]),
        "registers_per_thread": float(m["launch__registers_per_thread"]),
        "grid": float(m["launch__grid_size"]),
        "block": float(m["launch__block_size"]),
        "warps_active_pct": float(m["sm__warps_active.avg.pct_of_peak_sustained_active"]),
        "inst_executed": float(m["smsp__inst_executed.sum"]),
        "launch_list": f"profiles/launches_{rnd}_{cfg}.csv ({len(times)} sweep launches, mean "
                       f"{statistics.mean(times):.0f} us, median {statistics.median(times):.0f} us; "
                       "serialised, cold-cache)" if times else None,
        "round": rnd,
    }
    path = os.path.join(ROOT, "profiles", "ncu_sweep_summary.json")
    allc = json.load(open(path)) if os.path.exists(path) else {}
    allc[cfg] = summ
    json.dump(allc, open(path, "w"), indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()

"""Per-CUDA-line warp-stall samples of an ncu capture (cuda,sass source view):
python tools/ncu_lines.py REPORT.ncu-rep [TOP] [KERNEL_REGEX]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kfilter = ["--kernel-name", "regex:" + sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + kfilter,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines, fname, total = [], None, 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) >= 6 and r[0].isdigit():
        try:
            s = int(r[4])
        except ValueError:
            continue
        total += s
        lines.append((s, int(r[5]) if r[5].isdigit() else 0, fname, int(r[0]), r[1][:90]))
lines.sort(reverse=True)
print(f"total samples {total}")
for s, ni, f, ln, src in lines[:top]:
    print(f"{s:7d} {100 * s / max(total, 1):5.1f}% (not-issued {ni:6d}) {f}:{ln:<5d} {src}")

"""SASS instruction census of the library's kernels (cuobjdump -sass): counts of
the opcodes that prove the data path (UBLKCP = cp.async.bulk / 1-D TMA,
SYNCS = mbarrier, LDGSTS = cp.async, DFMA / DADD / DMUL fp64, LDS / STS,
SHFL, BAR, MEMBAR / FENCE, tcgen05 / UTMA* absent by design).
python tools/sass_census.py [LIB] > profiles/sass_census_r02.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2107_01745_b200", "lib", "libscenopt_b200.so")
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
OPS = ["UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "LDGSTS", "LDGDEPBAR", "DFMA", "DADD", "DMUL", "LDS", "STS",
       "LDG", "STG", "SHFL", "BAR", "MEMBAR", "FENCE", "ATOMG", "RED", "NANOSLEEP", "UTCMMA", "UTCBAR"]
func, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        func = m.group(1)
        counts[func] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
    if func and m:
        counts[func][m.group(1)] += 1


def short(f):
    m = re.search(r"_cu_[0-9a-f]{8}(\d+)", f) or re.search(r"N3scn(\d+)", f)
    if not m:
        return f[:28]
    k = int(m.group(1))
    name = f[m.end():m.end() + k]
    t = re.search(r"ILi(\d)ELi(\d)E", f[m.end() + k:])
    g = re.search(r"geom_(p\d)", f)  # sweep kernel geometry (four / six producer warps)
    return name + (f"<{t.group(1)},{t.group(2)}>" if t else "") + (f" {g.group(1)}" if g else "")


print(f"library: {os.path.relpath(lib, ROOT)}")
print(f"{'kernel':28s} {'total':>7s} " + " ".join(f"{o:>8s}" for o in OPS))
for f, c in counts.items():
    print(f"{short(f):28s} {sum(c.values()):7d} " + " ".join(f"{c.get(o, 0):8d}" for o in OPS))

"""Per-kernel count / mean / total of an ncu --metrics gpu__time_duration.sum
--csv launch list (cold-cache, serialised: shares, not absolutes).
python tools/launch_summary.py launches.csv [--last N]  (N = only the last N launches)"""
import collections, csv, sys

path = sys.argv[1]
last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else 0
hdr, rows = None, []
for r in csv.reader(open(path)):
    if "Kernel Name" in r:
        hdr = r
    elif hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((d["Kernel Name"].split("(")[0].replace("void ", "")[:48],
                         float(d["Metric Value"].replace(",", "")) / 1e3))
if last:
    rows = rows[-last:]
agg = collections.OrderedDict()
for k, t in rows:
    agg.setdefault(k, []).append(t)
tot = sum(t for _, t in rows)
print(f"{len(rows)} launches, {tot:.1f} us")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"  {k:48s} n={len(v):4d} mean={sum(v) / len(v):8.2f} us  total={sum(v):9.1f} us  {100 * sum(v) / tot:5.1f}%")

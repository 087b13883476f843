"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel and
grid shape, i.e. per multigrid level.  usage: python tools/ncu_levels.py launches.csv"""
import csv, re, sys, collections

rows = []
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"(k_\w+)(<[^(]*>)?", name)
    short = (m.group(1) + (m.group(2) or "")) if m else name[:40]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
          "msecond": 1e3}.get(unit, 1.0) * v
    rows.append((short, r["Grid Size"], r["Block Size"], us))
agg = collections.OrderedDict()
for k, g, b, us in rows:
    a = agg.setdefault((k, g, b), [0, 0.0])
    a[0] += 1
    a[1] += us
tot = sum(a[1] for a in agg.values())
print(f"| kernel | grid | block | launches | total us | mean us | share |")
print("|---|---|---|---|---|---|---|")
for (k, g, b), (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {g} | {b} | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
print(f"| **total** | | | {sum(a[0] for a in agg.values())} | {tot:.1f} | | 100% |")

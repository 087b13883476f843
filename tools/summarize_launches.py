"""Summarizes an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total and mean device time, share of the total."""
import csv
import collections
import re
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = i
            break
    h = rows[hdr]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= iv:
            continue
        try:
            v = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[iu], 1.0)
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("pmg::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{name}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
    lines.append(f"| **total** | {sum(a[0] for a in agg.values())} | {tot:.1f} | | 100% |")
    txt = "\n".join(lines)
    if out:
        open(out, "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main(*sys.argv[1:])

"""FP64 flops per node and DRAM bytes of the Give kernels from an ncu metrics CSV
(tools/r02_give.sh): writes profiles/give_flops.json and prints a table.
usage: python tools/give_flops.py <csv> <nr> <nt> <split> [out.json]"""
import collections
import csv
import json
import sys

path, nr, nt, split = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
h = rows[hdr]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= iv:
        continue
    key = (r[iid], r[ik].split("(")[0].replace("void ", "").replace("pmg::<unnamed>::", ""))
    per.setdefault(key, {})[r[im]] = float(r[iv].replace(",", ""))
nodes = {"residual": nr * nt, "circle": split * nt, "radial": (nr - split) * nt}
kind_of = lambda name: ("residual" if "apply" in name else "circle" if "circle" in name
                        else "radial" if "radial" in name else None)
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for (_, name), m in per.items():
    k = kind_of(name)
    if k is None:
        continue
    fl = (2 * m.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
          + m.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
          + m.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0))
    agg[k]["flops"] += fl
    agg[k]["dram"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    agg[k]["launches"] += 1
out = {}
print("| kernel | launches counted | FP64 flops / node | DRAM bytes / node |")
print("|---|---|---|---|")
for k, a in agg.items():
    # sweeps: one B + one W launch make a sweep over the region's nodes; the
    # capture may hold several repetitions -> normalise by launches
    per_launch_nodes = nodes[k] * (1.0 if k == "residual" else 0.5)
    fl = a["flops"] / (a["launches"] * per_launch_nodes)
    by = a["dram"] / (a["launches"] * per_launch_nodes)
    out[k] = round(fl, 1)
    print(f"| Give {k} | {int(a['launches'])} | {fl:.1f} | {by:.1f} |")
if len(sys.argv) > 5:
    json.dump(out, open(sys.argv[5], "w"), indent=1)

"""Aggregate an ncu --csv launch list (gpu__time_duration + dram bytes + L2 hit) per kernel name."""
import collections
import csv
import sys


def main(path, skip=0):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        if int(r[ii]) < skip:
            continue
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for d in per.values():
        name = d["name"].split("(")[0].replace("void ", "")[:60]
        a = agg[name]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0) / 1e6  # ns -> ms
        a[2] += (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e9
    tot = sum(a[1] for a in agg.values())
    print(f"total {tot:.1f} ms over {len(per)} launches")
    for name, a in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
        print(f"{a[1]:9.2f} ms {a[1] / tot * 100:5.1f}%  x{a[0]:<4d} dram {a[2]:8.2f} GB  {name}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)

"""Summarise an ncu --csv launch list (gpu__time_duration etc.) per kernel launch."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
tot = sum(v.get("gpu__time_duration.sum", 0) for v in d.values())
for k, v in d.items():
    t = v.get("gpu__time_duration.sum", 0)
    print(f"{v['name'][:64]:64s} {t / 1e3:8.1f}us {t / tot * 100:5.1f}% rd={v.get('dram__bytes_read.sum', 0) / 1e6:7.1f}MB "
          f"wr={v.get('dram__bytes_write.sum', 0) / 1e6:7.1f}MB inst={v.get('smsp__inst_executed.sum', 0) / 1e6:6.1f}M")
print(f"total {tot / 1e3:.1f} us")

if len(sys.argv) > 2 and sys.argv[2] == "--by-kernel":  # aggregate: launches, median, share
    import statistics
    agg = OrderedDict()
    for v in d.values():
        agg.setdefault(v["name"][:64], []).append(v.get("gpu__time_duration.sum", 0))
    print("\nper kernel: launches, median us, total us, share of all launches")
    for k, ts in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:64s} {len(ts):5d} {statistics.median(ts) / 1e3:9.1f} {sum(ts) / 1e3:10.1f} {sum(ts) / tot * 100:5.1f}%")

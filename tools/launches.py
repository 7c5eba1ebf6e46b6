"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ launch__grid_size])."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
ix = {k: i for i, k in enumerate(hdr)}
launch = collections.OrderedDict()
for r in rows[hdr_i + 1:]:
    if len(r) != len(hdr):
        continue
    d = launch.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
    d[r[ix["Metric Name"]]] = r[ix["Metric Value"]].replace(",", "")
items = list(launch.values())
last = int(sys.argv[2]) if len(sys.argv) > 2 else len(items)
tot = 0.0
for it in items[-last:]:
    t = float(it.get("gpu__time_duration.sum", 0))
    tot += t
    print(f"{it['name'][:70]:70s} grid={it.get('launch__grid_size', ''):>6s} {t / 1e3:9.1f} us")
print(f"total {tot / 1e3:.1f} us over {last} launches")

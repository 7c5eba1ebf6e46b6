"""Aggregate an ncu launch-list CSV by kernel family (second half = the profiled call)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
ix = {k: i for i, k in enumerate(hdr)}
L = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) != len(hdr):
        continue
    d = L.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
    d[r[ix["Metric Name"]]] = r[ix["Metric Value"]].replace(",", "")
items = list(L.values())
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
part = items[int(len(items) * (1 - frac)):]
keys = sys.argv[3].split(",") if len(sys.argv) > 3 else ["jacobi", "chol_kernel", "trsm_rows", "tc_gemm", "splitk",
                                                         "cheb", "ritz", "fill_omega", "signfix", "permute"]
agg = collections.defaultdict(lambda: [0, 0.0])
for it in part:
    n = it["name"]
    for key in keys:
        if key in n:
            n = key
            break
    agg[n][0] += 1
    agg[n][1] += float(it.get("gpu__time_duration.sum", 0))
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} n={v[0]:5d} total={v[1] / 1e3:9.1f}us avg={v[1] / v[0] / 1e3:8.1f}us")
print(f"total {tot / 1e3:.1f} us over {len(part)} launches")

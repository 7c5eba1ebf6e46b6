"""DRAM traffic of the tc_gemm launches of one contraction-only C4 move from an ncu CSV
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum on
tools/prof_move.py c4 inject): writes profiles/r02_traffic.json for bench.py's roofline."""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
H = rows[hi]
ix = {k: i for i, k in enumerate(H)}
L = {}
for r in rows[hi + 1:]:
    if len(r) != len(H):
        continue
    d = L.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
    v = r[ix["Metric Value"]].replace(",", "")
    unit = r[ix["Metric Unit"]] if "Metric Unit" in ix else ""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    try:
        d[r[ix["Metric Name"]]] = float(v) * (scale if "bytes" in r[ix["Metric Name"]] else 1)
    except ValueError:
        pass
tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in L.values() if "tc_gemm" in d["name"])
n = sum(1 for d in L.values() if "tc_gemm" in d["name"])
out = {"kernel": "tc_gemm", "config": "c4 contraction-only left move (isometries injected)",
       "dram_bytes_per_step": tot, "tc_gemm_launches": n,
       "how": "ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
              "on tools/prof_move.py c4 inject (one move), summed over its tc_gemm launches",
       "compulsory_bytes_note": "SURVEY 8(d): ~104 MB compulsory per move (inputs + 34 MB written); the rest is the "
                                "unfused X1..X5 round trips of the sequential chain"}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out))

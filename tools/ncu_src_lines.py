"""Per-CUDA-source-line warp-stall samples from `ncu -i rep --page source --csv --print-source cuda,sass`.
    python tools/ncu_src_lines.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
H = rows[hdr]
ismp = H.index("Warp Stall Sampling (All Samples)")
lines, cur, sass = {}, None, {}
for r in rows[hdr + 1:]:
    if len(r) <= ismp:
        continue
    if r[0]:
        if not r[0].isdigit():   # a further file/function section
            cur = None
            continue
        cur = (int(r[0]), r[1].strip()[:100])
        lines.setdefault(cur, 0)
        continue
    try:
        s = int(r[ismp] or 0)
    except ValueError:
        continue
    if cur is not None:
        lines[cur] += s
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        sass.setdefault(cur, {}).setdefault(op.split(".")[0], 0)
        sass[cur][op.split(".")[0]] += s
tot = sum(lines.values())
print("total samples", tot)
for k, v in sorted(lines.items(), key=lambda kv: -kv[1])[:top]:
    ops = sorted(sass.get(k, {}).items(), key=lambda kv: -kv[1])[:4]
    print(f"{100.0 * v / max(tot, 1):5.1f}%  L{k[0]:4d}  {k[1]:<100s} {ops}")

"""Summaries of ncu launch lists (`--metrics gpu__time_duration.sum[,launch__grid_size] --csv`):
  python tools/launch_summary.py families <bench_step.csv> <out.txt>   per-kernel-family shares of one bench step
  python tools/launch_summary.py list <launches.csv> <out.txt>         one line per launch"""
import collections
import csv
import sys

KEYS = ["jacobi_cluster", "jacobi_lsv", "chol_kernel", "trsm_rows", "tc_gemm", "splitk", "cheb", "ritz", "fill_omega",
        "signfix", "permute", "replace_cols", "scale_commit", "chol_"]


def load(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[hi]
    ix = {k: i for i, k in enumerate(H)}
    L = {}
    for r in rows[hi + 1:]:
        if len(r) != len(H):
            continue
        d = L.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})
        d[r[ix["Metric Name"]]] = r[ix["Metric Value"]].replace(",", "")
    return L


def main():
    mode, src, dst = sys.argv[1:4]
    L = load(src)
    with open(dst, "w") as out:
        if mode == "list":
            for d in L.values():
                out.write(f"{d['name'][:70]:70s} grid={d.get('launch__grid_size', '?'):>6s} "
                          f"{float(d.get('gpu__time_duration.sum', 0)) / 1000:9.1f} us\n")
            return
        agg = collections.defaultdict(lambda: [0, 0.0])
        for d in L.values():
            n = d["name"]
            for k in KEYS:
                if k in n:
                    n = k
                    break
            agg[n][0] += 1
            agg[n][1] += float(d.get("gpu__time_duration.sum", 0)) / 1000
        tot = sum(v[1] for v in agg.values())
        out.write("# ncu --profile-from-start off --metrics gpu__time_duration.sum: one timed step of `python bench.py "
                  "--steps 1 --warmup 3`\n# (CTM_BENCH_PROFILE=1). Serialised, cold-cache per-launch times; the step runs "
                  "its solver chains concurrently,\n# so the sum exceeds the step time. Share = kernel family time / sum.\n")
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            out.write(f"{k[:60]:60s} n={v[0]:6d} total={v[1]:10.1f}us share={100 * v[1] / tot:5.1f}%\n")
        out.write(f"total {tot:.1f} us over {len(L)} launches\n")


if __name__ == "__main__":
    main()

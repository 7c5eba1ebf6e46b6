"""Summarise an `ncu --set full` report (exported with `ncu -i X.ncu-rep --page raw --csv`)
into one line per profiled launch: duration, DMMA pipe utilisation, DRAM traffic,
occupancy, issue activity and the top stall reasons.

    ncu -i gpurun_out/prof.ncu-rep --page raw --csv > /tmp/raw.csv
    python tools/ncu_summary.py /tmp/raw.csv > profiles/rNN_ncu_<name>.txt
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur_us"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "dmma_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        out = [f"{r[ix['Kernel Name']][:60]} grid={r[ix['Grid Size']]} block={r[ix['Block Size']]}"]
        for k, name in KEYS:
            if k in ix:
                out.append(f"{name}={r[ix[k]]}{units[ix[k]] if units[ix[k]] not in ('', '%') else ''}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        out.append("stalls=" + ",".join(f"{n}:{v:.2f}" for v, n in stalls[:6]))
        print(" | ".join(out))


if __name__ == "__main__":
    main(sys.argv[1])

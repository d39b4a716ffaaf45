"""Top warp-stall reasons (and a few throughput counters) from
`ncu -i REPORT --page raw --csv` on stdin, one block per kernel."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
if len(rows) < 3:
    sys.exit("no data")
head = rows[0]
for r in rows[2:]:
    name = r[head.index("Kernel Name")][:100]
    print(f"== {name}")
    vals = {}
    for h, v in zip(head, r):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                vals[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
            except ValueError:
                pass
    tot = sum(vals.values()) or 1.0
    for k, v in sorted(vals.items(), key=lambda kv: -kv[1])[:8]:
        print(f"   stall {k:28s} {v:8.2f}  ({100 * v / tot:4.1f}%)")
    for h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"):
        if h in head:
            print(f"   {h:60s} {r[head.index(h)]}")

"""Condense an `ncu --set full` report of the Ax kernel into profiles/."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "gpc__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main(rep, out_txt, out_json, title):
    h, units, v = raw(rep)
    d = {k: (x, u) for k, u, x in zip(h, units, v)}
    stalls = {}
    for k, (x, _) in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                if float(x) > 0:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(x)
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    name = d.get("Kernel Name", ("?", ""))[0]
    lines = [f"# {title}", f"kernel: {name}"]
    for k in KEYS:
        if k in d:
            lines.append(f"{k:70s} {d[k][0]:>16s} {d[k][1]}")
    lines.append("stall reasons (share of PC samples):")
    for k, x in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]:
        lines.append(f"  {k:40s} {x / tot:6.1%}")
    open(out_txt, "w").write("\n".join(lines) + "\n")
    mb = lambda k: float(d[k][0].replace(",", "")) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}[d[k][1]]
    summary = {"kernel": name, "source": rep,
               "duration_us": float(d["gpu__time_duration.sum"][0]),
               "dram_bytes_per_launch": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
               "dram_read_bytes": mb("dram__bytes_read.sum"),
               "dram_write_bytes": mb("dram__bytes_write.sum")}
    json.dump(summary, open(out_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:5])

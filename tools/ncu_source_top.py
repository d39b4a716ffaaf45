"""Top source lines (or SASS instructions) by warp-stall samples from
`ncu -i REPORT --page source --csv [--print-source cuda|sass]` on stdin."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
# the CSV may hold several kernels / files: find header rows
out = []
head = None
for r in rows:
    if r and ("Warp Stall Sampling (All Samples)" in r or "Source" in r[:3]):
        if "Warp Stall Sampling (All Samples)" in r:
            head = r
            continue
    if head is None or len(r) != len(head):
        continue
    try:
        samp = float(r[head.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    src = r[head.index("Source")] if "Source" in head else r[1]
    line = r[head.index("#")] if "#" in head else ""
    out.append((samp, line, src.strip()[:110]))
tot = sum(s for s, _, _ in out) or 1.0
print(f"# columns: {head[:12] if head else None}")
for s, line, src in sorted(out, reverse=True)[:int(sys.argv[1]) if len(sys.argv) > 1 else 30]:
    print(f"{100 * s / tot:5.1f}%  {line:>5}  {src}")

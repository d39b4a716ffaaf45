"""Per-instruction warp-stall attribution from `ncu -i R --page source --csv
--print-source sass`: top instructions with their dominant stall reasons, and
totals per opcode."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
head = rows[hi]
S = head.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h) for i, h in enumerate(head) if h.startswith("stall_") and "Not Issued" not in h]
items = []
for r in rows[hi + 1:]:
    if len(r) != len(head):
        continue
    try:
        s = float(r[S] or 0)
    except ValueError:
        continue
    rs = sorted(((float(r[i] or 0), h[6:]) for i, h in reasons), reverse=True)[:3]
    items.append((s, r[0], r[1].strip(), rs))
tot = sum(x[0] for x in items) or 1
print(f"total samples {tot:.0f}")
for s, a, src, rs in sorted(items, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    why = ", ".join(f"{n} {100 * v / s:.0f}%" for v, n in rs if v > 0) if s else ""
    print(f"{100 * s / tot:5.1f}%  {a}  {src[:48]:48s} {why}")
byop = defaultdict(float)
byreason = defaultdict(float)
for s, a, src, rs in items:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    byop[op.split(".")[0]] += s
for r in rows[hi + 1:]:
    if len(r) != len(head):
        continue
    for i, h in reasons:
        try:
            byreason[h[6:]] += float(r[i] or 0)
        except ValueError:
            pass
print("by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(byop.items(), key=lambda kv: -kv[1])[:12]))
print("by reason:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(byreason.items(), key=lambda kv: -kv[1])[:10]))

"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, title):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        val = float(r[ix["Metric Value"]].replace(",", "")) * SCALE[r[ix["Metric Unit"]]]
        agg[r[ix["Kernel Name"]].split("(const")[0].split("(double")[0][:80]].append(val)
    tot = sum(sum(v) for v in agg.values())
    print(f"# {title}")
    print("# gpu__time_duration.sum, --clock-control none: cold-cache serialised launches, compare SHARES")
    print(f"{'kernel':80s} {'launches':>8s} {'mean_us':>9s} {'median_us':>9s} {'share':>7s}")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        med = sorted(v)[len(v) // 2]
        print(f"{k:80s} {len(v):8d} {sum(v) / len(v):9.2f} {med:9.2f} {sum(v) / tot:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])

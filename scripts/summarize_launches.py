"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel shares.

    python scripts/summarize_launches.py gpurun_out/launches.csv [--md]
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("wsb::", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return name[:70]


def main():
    path = sys.argv[1]
    md = "--md" in sys.argv
    rows = []
    hdr = None
    with open(path) as f:
        for r in csv.reader(f):
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                if d.get("Metric Name") == "gpu__time_duration.sum":
                    v = float(d["Metric Value"].replace(",", ""))
                    unit = d.get("Metric Unit", "ns")
                    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
                    full = d["Kernel Name"]
                    tmpl = re.search(r"<(\d+), *(\d+)>", full)
                    key = short(full) + (f"<{tmpl.group(1)},{tmpl.group(2)}>" if tmpl else "")
                    rows.append((key, v * scale, d.get("Grid Size", "")))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, us, _ in rows:
        agg[k][0] += 1
        agg[k][1] += us
    total = sum(v[1] for v in agg.values())
    items = sorted(agg.items(), key=lambda kv: -kv[1][1])
    if md:
        print(f"{len(rows)} launches, {total / 1e3:.2f} ms total device time (serialised, cold-cache under ncu)\n")
        print("| kernel | launches | total µs | mean µs | share |")
        print("|---|---:|---:|---:|---:|")
        for k, (n, us) in items:
            print(f"| `{k}` | {n} | {us:.0f} | {us / n:.1f} | {100 * us / total:.1f}% |")
    else:
        for k, (n, us) in items:
            print(f"{100 * us / total:6.2f}%  {n:6d}  {us:12.1f} us  {k}")


if __name__ == "__main__":
    main()

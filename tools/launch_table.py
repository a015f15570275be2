"""Launch-list table (markdown) from an `ncu --metrics gpu__time_duration.sum --csv` log.
Usage: python tools/launch_table.py launches.csv [title] > profiles/<round>_launches.md"""
import collections
import csv
import sys


def main(path, title="Launch list"):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ki].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
    total = sum(v[1] for v in agg.values())
    print(f"# {title}\n")
    print("Cold-cache, serialised per-launch times: compare shares, not absolutes.\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if ms / total < 0.002:
            continue
        print(f"| `{name}` | {n} | {ms:.2f} | {100 * ms / total:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))

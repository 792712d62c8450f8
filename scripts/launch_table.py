"""Markdown table of an ncu launch list (--metrics gpu__time_duration.sum --csv).
Usage: python scripts/launch_table.py launches.csv > profiles/rN_launches.md"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    t = collections.defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            t[name].append(float(r[vi].replace(",", "")) / 1000.0)
    ours = sum(sum(v) for k, v in t.items() if "rtgs::" in k)
    print("| kernel | launches | mean µs | min µs | max µs | share of librtgs time |")
    print("|---|---|---|---|---|---|")
    for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
        share = f"{sum(v) / ours:.3f}" if "rtgs::" in k else "(torch)"
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.2f} | {min(v):.2f} | {max(v):.2f} | {share} |")


if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into a
markdown table (launches, serialised ms and share per kernel).

    python tools/launch_list.py gpurun_out/x.csv "title" [--skip-before KERNEL N] > profiles/x.md
"""
import csv
import re
import sys
from collections import OrderedDict


def main():
    path, title = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").strip()
        name = re.sub(r"irisgpu::(\(anonymous namespace\)::)?", "", name)
        ns = float(r[vi].replace(",", ""))
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + ns / 1e6)
    tot = sum(t for _, t in agg.values())
    print(f"# {title}")
    print("# (ncu --metrics gpu__time_duration.sum --clock-control none; serialised, cold-cache: compare SHARES,"
          " not absolutes)\n")
    print("| kernel | launches | ms (serialised) | share |\n|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {n} | {t:.2f} | {100 * t / tot:.1f}% |")
    print(f"| total | {sum(n for n, _ in agg.values())} | {tot:.1f} | 100% |")


if __name__ == "__main__":
    main()

"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/ncu_launches.py gpurun_out/launches.csv > profiles/r01_launches.md

Launch times under ncu are serialised and cold-cache, so compare SHARES of the step
with bench.py's live CUDA-event numbers, not absolute times.
"""
import collections
import csv
import re
import sys


def short(name):
    name = re.sub(r"\(.*\)$", "", name)                 # drop the parameter list
    name = name.replace("rp::k::", "").replace("rp::", "").replace("(anonymous namespace)::", "")
    name = name.replace("<unnamed>::", "")
    return name


def main(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
        rows.append((short(r["Kernel Name"]), r["Grid Size"], r["Block Size"], us))
    tot = collections.OrderedDict()
    for name, grid, block, us in rows:
        t = tot.setdefault(name, [0, 0.0, grid, block])
        t[0] += 1
        t[1] += us
    total = sum(t[1] for t in tot.values())
    print(f"# ncu launch list summary: {path}\n")
    print(f"{len(rows)} launches, {total / 1e3:.3f} ms total (serialised, cold-cache under ncu)\n")
    print("| kernel | launches | total ms | mean us | share | grid | block |")
    print("|---|---|---|---|---|---|---|")
    for name, (n, us, grid, block) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{name}` | {n} | {us / 1e3:.3f} | {us / n:.1f} | {100 * us / total:.1f}% | {grid} | {block} |")


if __name__ == "__main__":
    main(sys.argv[1])

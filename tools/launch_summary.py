"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: total
ms, share, launches and mean us per kernel.

    python tools/launch_summary.py launches.csv [name_width] [--skip-first]

--skip-first drops the first gemm_dmma launch (bench.py's input-generation
SYRK, which precedes the timed factorizations)."""
import collections
import csv
import sys

args = [a for a in sys.argv[1:] if not a.startswith("--")]
skip_first = "--skip-first" in sys.argv
width = int(args[1]) if len(args) > 1 else 70
d = collections.defaultdict(lambda: [0, 0.0])
h = None
for r in csv.reader(open(args[0])):
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        x = dict(zip(h, r))
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        if skip_first and "gemm_dmma" in x["Kernel Name"]:
            skip_first = False
            continue
        v = float(x["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(x["Metric Unit"], 1.0)
        k = x["Kernel Name"][:width]
        d[k][0] += 1
        d[k][1] += v
tot = sum(v[1] for v in d.values())
print(f"total {tot / 1e3:.2f} ms over {sum(v[0] for v in d.values())} launches (cold-cache, serialised by ncu)")
for k, v in sorted(d.items(), key=lambda t: -t[1][1])[:15]:
    print(f"{v[1] / 1e3:9.2f} ms {100 * v[1] / tot:5.1f}% {v[0]:5d} {v[1] / v[0]:10.1f} us  {k}")

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: total
ms, share, launches and mean us per kernel."""
import collections
import csv
import sys

d = collections.defaultdict(lambda: [0, 0.0])
h = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        h = r
        continue
    if h and len(r) == len(h):
        x = dict(zip(h, r))
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(x["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(x["Metric Unit"], 1.0)
        k = x["Kernel Name"][: int(sys.argv[2]) if len(sys.argv) > 2 else 70]
        d[k][0] += 1
        d[k][1] += v
tot = sum(v[1] for v in d.values())
print(f"total {tot / 1e3:.2f} ms over {sum(v[0] for v in d.values())} launches")
for k, v in sorted(d.items(), key=lambda t: -t[1][1])[:15]:
    print(f"{v[1] / 1e3:9.2f} ms {100 * v[1] / tot:5.1f}% {v[0]:5d} {v[1] / v[0]:10.1f} us  {k}")

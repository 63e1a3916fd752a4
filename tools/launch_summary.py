"""Summarise an ncu --metrics gpu__time_duration.sum launch list (skips the
input-generation SYRK, the first TMA launch, when asked)."""
import collections
import csv
import sys

path = sys.argv[1]
skip_first = "--skip-first" in sys.argv
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt, mx = collections.defaultdict(float), collections.Counter(), collections.defaultdict(float)
first = skip_first
for r in rows[hdr_i + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", "")) / 1e6
    name = r[ki].split("(")[0][:80]
    if first and "gemm_dmma" in name:
        first = False
        continue
    tot[name] += v
    cnt[name] += 1
    mx[name] = max(mx[name], v)
T = sum(tot.values())
print(f"{'ms':>9} {'share':>6} {'launches':>8} {'max ms':>8}  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"{v:9.2f} {100 * v / T:5.1f}% {cnt[k]:8d} {mx[k]:8.3f}  {k}")
print(f"{T:9.2f}  total over {sum(cnt.values())} launches (cold-cache, serialised by ncu)")

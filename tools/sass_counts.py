"""Per-kernel SASS instruction counts that prove the hardware path
(UTMALDG = TMA load, DMMA = FP64 tensor MMA, UTC*MMA = tcgen05.mma, LDTM/STTM =
tcgen05.ld/st, REDG = red.global, LDGSTS = cp.async) for the built library.

    python tools/sass_counts.py [lib.so] > profiles/r02_sass_counts.txt
"""
from __future__ import annotations

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "paper_2604_07311_b200" / "_lib" / "libblockfam_b200.so"
KEYS = ["UTMALDG", "UTMASTG", "UTMAREDG", "DMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "DFMA", "REDG", "LDGSTS",
        "SYNCS"]

sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
counts: dict[str, collections.Counter] = collections.defaultdict(collections.Counter)
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,6}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur:
        counts[cur][m.group(1)] += 1
names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# SASS instruction counts per kernel: {LIB.name} (cuobjdump -sass, sm_100a)")
print("# kernel | " + " ".join(KEYS))
for (fn, c), name in sorted(zip(counts.items(), names), key=lambda x: x[1]):
    sel = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
    if sel:
        print(f"{name[:150]} | {sel}")

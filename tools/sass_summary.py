"""Per-kernel SASS instruction-class summary of the built library (cuobjdump -sass).

    python tools/sass_summary.py [lib.so] > profiles/r02/sass_summary.txt
Counts, per kernel, the instructions that show which hardware path it uses: DMMA (FP64 tensor
core), UTCHMMA / UTCBAR / LDTM / STTM (tcgen05 tensor core + TMEM), UTMALDG / UBLKCP (TMA tensor /
bulk copies), LDGSTS (Ampere cp.async), SYNCS (mbarrier), DFMA / DMUL / DADD (FP64 CUDA cores),
F2F (conversions), LDS / STS / LDG / STG / RED (memory).
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1911_03813_b200/_lib/libmomentcp_b200.so"
CLASSES = ["DMMA", "UTCHMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "UTMAPF", "LDGSTS",
           "SYNCS", "DFMA", "DMUL", "DADD", "F2F", "LDS", "STS", "LDG", "STG", "RED", "ATOMS",
           "BAR"]
out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
kern = None
counts = collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m:
        op = m.group(2)
        for c in CLASSES:
            if op == c or op.startswith(c + "."):
                counts[kern][c] += 1
dem = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout
names = dem.splitlines()
print(f"# SASS instruction classes per kernel: {LIB}")
print("# columns: " + " ".join(CLASSES))
for (k, c), name in zip(counts.items(), names):
    if not any(c.values()):
        continue
    short = re.sub(r"\(.*", "", name)[:70]
    print(f"{short:70s} " + " ".join(f"{c[x]:5d}" for x in CLASSES))

"""Per-kernel SASS instruction summary of libtt_hotpath.so (cuobjdump -sass): counts of the
FP64 tensor-core (DMMA), TMA (UTMALDG / UBLKCP), shared-memory (LDS / STS), global (LDG / STG,
incl. the 256-bit STG.E.ENL2.256) and FP64 FMA (DFMA) instructions, plus registers / shared
memory from cuobjdump -res-usage.  Usage: python tools/sass_summary.py [lib] > out.txt"""
import collections
import os
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2509_11890_b200", "libtt_hotpath.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
usage = {}
cur = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        cur = m.group(1)
    m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
    if m and cur:
        usage[cur] = (int(m.group(1)), int(m.group(2)))
pats = collections.OrderedDict([
    ("DMMA", r"\bDMMA\."), ("HMMA/UTC", r"\b(HMMA|UTCHMMA|UTCQMMA)"), ("UTMALDG", r"\bUTMALDG"),
    ("UBLKCP", r"\bUBLKCP"), ("LDGSTS", r"\bLDGSTS"), ("LDS", r"\bLDS\b|\bLDS\."),
    ("LDS.128", r"\bLDS\.128"), ("LDSM", r"\bLDSM"),
    ("STS", r"\bSTS\b|\bSTS\."), ("LDG", r"\bLDG\."), ("STG", r"\bSTG\."), ("STG.256", r"STG\.E[^ ]*\.256"),
    ("DFMA", r"\bDFMA\b"), ("SYNCS", r"\bSYNCS\."), ("BAR", r"\bBAR\."), ("ATOM/RED", r"\b(ATOMG|RED)\."),
])
kern = None
counts = collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None or not re.search(r"/\*[0-9a-f]{4}\*/", line):
        continue
    for k, p in pats.items():
        if re.search(p, line):
            counts[kern][k] += 1
demangle = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
tot = collections.Counter()
print(f"{'kernel':70s} {'REG':>4s} {'SMEM':>6s} " + " ".join(f"{k:>8s}" for k in pats))
for (k, c), name in sorted(zip(counts.items(), demangle), key=lambda x: -x[0][1]["DMMA"]):
    tot.update(c)
    reg, sm = usage.get(k, (0, 0))
    short = re.sub(r"\s+", "", name)[:70]
    print(f"{short:70s} {reg:4d} {sm:6d} " + " ".join(f"{c[p]:8d}" for p in pats))
print(f"{'TOTAL (' + str(len(counts)) + ' kernels)':70s} {'':4s} {'':6s} " + " ".join(f"{tot[p]:8d}" for p in pats))

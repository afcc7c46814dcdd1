"""Print registers / stack per GEMM kernel instantiation of the built library."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2509_11890_b200/libtt_hotpath.so"
out = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True).stdout
lines = out.splitlines()
for i, l in enumerate(lines):
    m = re.search(r"Function (\S+):", l)
    if not m or i + 1 >= len(lines):
        continue
    name = m.group(1)
    r = re.search(r"REG:(\d+) STACK:(\d+)", lines[i + 1])
    t = re.search(r"dmma_gemm_(v\d)_kernelI(.*)E", name)
    if t and r:
        args = re.findall(r"L([bi])(\d+)E", t.group(2))
        print(t.group(1), ",".join(v for _, v in args), "REG", r.group(1), "STACK", r.group(2))

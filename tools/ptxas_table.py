"""Compile one csrc/*.cu with -Xptxas -v and print registers / spills per kernel (matching a regex)."""
import re
import subprocess
import sys

src, pat = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else ".")
defs = ["-D" + d for d in sys.argv[3:]]
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                      "-Xptxas", "-v", *defs, "-I", "include", "-c", src, "-o", "/tmp/_ptxas.o"],
                     capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        rows.setdefault(cur, ["", ""])
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows[cur][1] = "spill %s/%s" % m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows[cur][0] = "%s regs" % m.group(1)
for k, (r, sp) in rows.items():
    d = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"\(anonymous namespace\)::|\(.*", "", d)
    if re.search(pat, d):
        print("%-60s %-10s %s" % (d, r, sp))

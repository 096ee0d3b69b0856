"""Per-kernel register / spill differences between two build directories
(ptxas -v logs):  python tools/spill_diff.py _build _build_old"""
import glob
import re
import subprocess
import sys


def parse(d):
    out = {}
    for f in glob.glob(d + "/*.log"):
        fn = None
        for line in open(f):
            m = re.search(r"Compiling entry function '(\S+)'", line)
            if m:
                fn = m.group(1)
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m and fn:
                out.setdefault(fn, {})["spill"] = (int(m.group(1)), int(m.group(2)))
            m = re.search(r"Used (\d+) registers", line)
            if m and fn:
                out.setdefault(fn, {})["regs"] = int(m.group(1))
    return out


a, b = parse(sys.argv[1]), parse(sys.argv[2])
for k in sorted(a):
    if a[k] != b.get(k):
        n = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
        print(a[k], "vs", b.get(k), n[:120])

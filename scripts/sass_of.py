"""Prints the SASS of the kernels of a built object whose mangled name contains a substring:
python scripts/sass_of.py build/bound_v3.o k1v3_kernelILi8 [--grep REGEX]"""
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
rx = re.compile(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[3] == "--grep" else None
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
on = False
for line in out.splitlines():
    if line.strip().startswith("Function :"):
        on = pat in line
        if on:
            print(line)
        continue
    if on and (rx is None or rx.search(line)):
        print(line)

"""Extract one kernel's SASS from a shared library (dev tool).
usage: sass_fn.py LIB SUBSTRING  -> prints the first function whose name contains SUBSTRING"""
import subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
blocks = out.split("\t\tFunction : ")
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if sys.argv[2] in name:
        print(name)
        print(b)
        break

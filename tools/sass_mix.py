"""Opcode histogram of one kernel's SASS (cuobjdump -sass), optionally restricted to its hottest loop.

    python tools/sass_mix.py <lib.so> <function-name-substring>
"""
import collections
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", f)
    c = collections.Counter(o for o in ops)
    print(name, len(ops))
    print("  ", ", ".join(f"{k}:{v}" for k, v in c.most_common(24)))

"""Per-pair instruction counts of a pair kernel's innermost loop(s) containing MUFU.RSQ64H (one per pair).

    python tools/sass_loop.py <lib.so> <function-substring>
Prints, for each innermost loop with MUFU.RSQ64H: pairs per iteration, FP64 (DFMA/DMUL/DADD) and other instructions
per pair, and the issue-model cycles per warp-pair 2*FP64 + other.
"""
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", out)[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = []
    for ln in f.splitlines():
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", ln)
        if m:
            ops.append((int(m.group(1), 16), m.group(3), m.group(4)))
    loops = []
    for addr, op, args in ops:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", args)
            if t and int(t.group(1), 16) < addr:
                lo = int(t.group(1), 16)
                body = [o for o in ops if lo <= o[0] <= addr]
                if any(o[1].startswith("MUFU.RSQ64H") for o in body):
                    loops.append((lo, addr, body))
    # innermost: no other MUFU-loop strictly inside
    inner = [L for L in loops if not any(M is not L and L[0] <= M[0] and M[1] <= L[1] for M in loops)]
    print(name)
    for lo, hi, body in inner:
        npair = sum(1 for o in body if o[1].startswith("MUFU.RSQ64H"))
        fp = sum(1 for o in body if o[1] in ("DFMA", "DMUL", "DADD"))
        oth = len(body) - fp
        print(f"  loop {lo:#x}-{hi:#x}: {npair} pairs/iter, FP64 {fp / npair:.2f}/pair, other {oth / npair:.2f}/pair, "
              f"issue-model {(2 * fp + oth) / npair:.1f} cycles/warp-pair")

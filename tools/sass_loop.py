"""Per-pair instruction counts of a pair kernel's innermost loop(s) containing MUFU.RSQ64H or MUFU.RSQ (one per pair).

    python tools/sass_loop.py <lib.so> <function-substring>
Prints, for each innermost loop with MUFU.RSQ(64H): pairs per iteration, FP64 (DFMA/DMUL/DADD) and other instructions
per pair, and the issue-model cycles per warp-pair 2*FP64 + other.
"""
import re
import subprocess
import sys


def loops(lib, pat):
    """[(function, [(pairs_per_iter, fp64_per_pair, other_per_pair), ...])] for functions whose name contains pat."""
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    res = []
    for f in re.split(r"\n\s+Function : ", out)[1:]:
        name = f.split("\n", 1)[0].strip()
        if pat in name:
            res.append((name, _inner_loops(f)))
    return res


def _inner_loops(f):
    ops = []
    for ln in f.splitlines():
        m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)([^;]*);", ln)
        if m:
            ops.append((int(m.group(1), 16), m.group(3), m.group(4)))
    found = []
    for addr, op, args in ops:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", args)
            if t and int(t.group(1), 16) < addr:
                lo = int(t.group(1), 16)
                body = [o for o in ops if lo <= o[0] <= addr]
                if any(o[1].startswith("MUFU.RSQ") for o in body):
                    found.append((lo, addr, body))
    # innermost: no other MUFU-loop strictly inside
    inner = [L for L in found if not any(M is not L and L[0] <= M[0] and M[1] <= L[1] for M in found)]
    res = []
    for lo, hi, body in inner:
        npair = sum(1 for o in body if o[1].startswith("MUFU.RSQ"))
        fp = sum(1 for o in body if o[1] in ("DFMA", "DMUL", "DADD"))
        res.append((npair, fp / npair, (len(body) - fp) / npair))
    return res


def main_loop(lib, pat):
    """(fp64_per_pair, other_per_pair) of the innermost pair loop with the most pairs per iteration, or None."""
    best = None
    for _, ls in loops(lib, pat):
        for npair, fp, oth in ls:
            if best is None or npair > best[0]:
                best = (npair, fp, oth)
    return None if best is None else best[1:]


if __name__ == "__main__":
    for name, ls in loops(sys.argv[1], sys.argv[2]):
        print(name)
        for npair, fp, oth in ls:
            print(f"  {npair} pairs/iter, FP64 {fp:.2f}/pair, other {oth:.2f}/pair, "
                  f"issue-model {2 * fp + oth:.1f} cycles/warp-pair")

"""Per-region instruction / stall-sample profile of one kernel from an ncu report (SASS source page).

    python tools/ncu_sass_profile.py <prof.ncu-rep> [top] [kernel-name-substring]
Prints the loops (backward branches) with their executed warp instructions and stall samples, and the top
instructions by samples.
"""
import csv
import io
import re
import subprocess
import sys


def rows(rep, kernel=None):
    """SASS rows of the first captured kernel whose name contains `kernel` (default: the first kernel)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    lines = out.splitlines()
    starts = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
    sec = 0
    if kernel:
        sec = [k for k in range(len(starts) - 1) if kernel in lines[starts[k]]][0]
    lines = lines[starts[sec] + 1:starts[sec + 1]]
    hi = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
    rd = list(csv.reader(io.StringIO("\n".join(lines[hi:]))))
    h = rd[0]
    ia, isrc, isamp, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    res = []
    for r in rd[1:]:
        if len(r) <= iex:
            continue
        try:
            res.append((int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iex] or 0)))
        except ValueError:
            pass
    return res


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    R = rows(rep, sys.argv[3] if len(sys.argv) > 3 else None)
    base = R[0][0]
    tot_s = sum(r[2] for r in R)
    tot_i = sum(r[3] for r in R)
    print(f"total samples {tot_s}, warp instructions {tot_i:.4g}")
    loops = []
    for a, src, s, n in R:
        m = re.match(r"(@!?U?P\w+\s+)?BRA\S*\s+(?:`\(\.L_x_\d+\)\s*)?(0x[0-9a-f]+)?", src)
        if src.split()[0].startswith("BRA") or (m and "BRA" in src):
            t = re.search(r"0x([0-9a-f]+)", src)
            if t:
                tgt = int(t.group(1), 16)
                tgt = tgt + base if tgt < base else tgt
                if tgt < a:
                    loops.append((tgt, a))
    for lo, hi in loops:
        body = [r for r in R if lo <= r[0] <= hi]
        s = sum(r[2] for r in body)
        n = sum(r[3] for r in body)
        if n > 0.01 * tot_i or s > 0.01 * tot_s:
            print(f"loop {lo - base:#x}-{hi - base:#x}: {len(body)} instrs, {n / tot_i:6.1%} of executed, {s / tot_s:6.1%} of samples")
    print("top instructions by samples:")
    for a, src, s, n in sorted(R, key=lambda r: -r[2])[:top]:
        print(f"  {a - base:#07x} {s:7d} {n:12d}  {src[:70]}")


if __name__ == "__main__":
    main()

"""Summarise ncu output for profiles/ (run here, on the CPU box, after gpurun brought the files back).

    python tools/ncu_summary.py launches <launches.csv> [steps]     -> per-kernel share of device time
    python tools/ncu_summary.py full <prof.ncu-rep> <out.json>       -> key metrics + stall mix of each captured launch

The launch list is cold-cache and serialised (ncu replays), so compare SHARES, not absolute times.
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, steps=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    out = []
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append({"kernel": n, "launches": c, "ms": v / 1e6, "share": v / tot})
    return {"total_ms": tot / 1e6, "kernels": out}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_static",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]


def full(rep, out_json):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = {"kernel": d[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                rec[k] = d[h.index(k)] + " " + units[h.index(k)]
        stalls = {}
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    v = float(d[h.index(k)])
                except ValueError:
                    continue
                if v > 0.01:
                    stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        rec["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
        try:
            rd = float(d[h.index("dram__bytes_read.sum")])
            wr = float(d[h.index("dram__bytes_write.sum")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rec["dram_bytes_total"] = rd * scale[units[h.index("dram__bytes_read.sum")]] + \
                wr * scale[units[h.index("dram__bytes_write.sum")]]
        except (ValueError, KeyError):
            pass
        res.append(rec)
    json.dump(res, open(out_json, "w"), indent=1)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        r = launches(sys.argv[2])
        steps = int(sys.argv[3]) if len(sys.argv) > 3 else None
        for k in r["kernels"]:
            per = f"  {k['ms'] / steps:9.3f} ms/step" if steps else ""
            print(f"{k['launches']:6d} {k['ms']:11.3f} ms {100 * k['share']:6.2f}%{per}  {k['kernel']}")
        print(f"total {r['total_ms']:.3f} ms")
    else:
        for rec in full(sys.argv[2], sys.argv[3]):
            print(json.dumps(rec))

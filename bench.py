"""bench.py -- GMRES matvecs/s (and time-to-solution) of the multiple-scattering matvec on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--mode direct|hier] [--impl nc|reference]

A "step" is one full matvec (I + A_off) x over all N patches (all of SURVEY.md §8(a)'s matvec rows), with
inputs resident in HBM.  N > 1 runs under torchrun, one rank per GPU, target patches sharded, one NCCL
all-gather per matvec (strong scaling: the layout is fixed).  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, the deliberately slow reference of this tier) on the box's
host cores on a bounded sample of the same workload (sampled target patches), on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "r02h_fp64_peak.txt")   # clocks during it: r02h_fp64_peak_clocks.csv


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--mode", default=None, choices=["direct", "hier"],
                    help="default: hier for C3-C5, direct for C1-C2")
    ap.add_argument("--impl", default="nc", choices=["nc", "reference"])
    ap.add_argument("--tables", default="physical", choices=["synthetic", "physical"])
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="target patches in the oracle sample (0 = auto)")
    ap.add_argument("--field-points", type=int, default=16384,
                    help="NEXT-3 sweep: points on the sphere of radius 1 -+ eps/5 (nc_field_near)")
    return ap.parse_args()


def load_fp64_peak():
    best = {}
    try:
        for line in open(FP64_PEAK_FILE):
            line = line.strip()
            if line.startswith("{") and '"kind"' in line:
                d = json.loads(line)
                best[d["kind"]] = max(best.get(d["kind"], 0.0), d["tflops"])
    except OSError:
        pass
    return best


# ncu --set full captures of the dominant kernel (tools/ncu_summary.py full), keyed by (kernel, config, mode)
TRAFFIC_PROFILES = {("k_pairs_grid", "C5", "hier"): "profiles/r05o_ncu_full_pairs_grid.json"}


def profiled_traffic(kernel, config, mode):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu capture, or (None, None)."""
    rel = TRAFFIC_PROFILES.get((kernel, config, mode))
    if not rel:
        return None, None
    try:
        for rec in json.load(open(os.path.join(ROOT, rel))):
            if kernel in rec.get("kernel", "") and rec.get("dram_bytes_total"):
                return float(rec["dram_bytes_total"]), rel
    except (OSError, ValueError):
        pass
    return None, None


def profiled_shared_wavefronts(kernel, config, mode, sms=148):
    """The second bound of the grid kernel: shared-memory load wavefronts per SM-cycle (the L1 data
    pipe retires one per cycle) and the share of them that are bank-conflict replays, from the committed capture."""
    rel = TRAFFIC_PROFILES.get((kernel, config, mode))
    if not rel:
        return None
    try:
        for rec in json.load(open(os.path.join(ROOT, rel))):
            if kernel not in rec.get("kernel", ""):
                continue
            num = lambda k: float(str(rec[k]).split()[0])
            wf = num("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum")
            cf = num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum")
            cycles = num("gpu__time_duration.sum") * 1e-3 * num("sm__cycles_elapsed.avg.per_second") * 1e9 * sms
            return {"shared_ld_wavefronts_per_sm_cycle": wf / cycles, "bank_conflict_share": cf / wf,
                    "source": rel + " (ncu capture, not this run)"}
    except (OSError, ValueError, KeyError):
        pass
    return None


def make_tables(cfg, which):
    from nc_inputs import synthetic_tables
    if which == "physical":
        from nc_inputs.tables import load_tables
        path = os.path.join(ROOT, "tables", "data", f"{cfg.name}.npz")
        return load_tables(path)
    return synthetic_tables(cfg.kind, cfg.eps, seed=4242)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_sample(cfg, tab, x, n_rows, seed=0):
    """Time the oracle on n_rows sampled target patches; returns (seconds, rows, threads)."""
    from oracle import oracle as O
    c = cfg.centers()
    rows = np.sort(np.random.default_rng(seed).choice(cfg.N, n_rows, replace=False))
    O.lib()
    t0 = time.perf_counter()
    O.matvec(cfg.kind, c, tab, x, rows=rows)
    return time.perf_counter() - t0, rows, O.num_threads()


def auto_sample_rows(cfg, tab, target_s=12.0):
    # calibrate with a 1-patch run, then size the sample to ~target_s of CPU work
    from nc_inputs import random_coeffs
    x = random_coeffs(cfg.N, tab.K, 2000 + int(cfg.name[1:]))
    t1, _, _ = cpu_oracle_sample(cfg, tab, x, 1)
    return int(max(1, min(cfg.N, round(target_s / max(t1, 1e-4)))))


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on the host cores, bounded samples."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from nc_inputs import CONFIGS, random_coeffs
    cfg = CONFIGS[args.config]
    tab = make_tables(cfg, args.tables)
    x = random_coeffs(cfg.N, tab.K, 2000 + int(cfg.name[1:]))
    n_rows = args.cpu_sample or auto_sample_rows(cfg, tab, target_s=8.0)
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_oracle_sample(cfg, tab, x, max(1, n_rows // 8))
    times = []
    for k in range(args.steps):
        t, rows, thr = cpu_oracle_sample(cfg, tab, x, n_rows, seed=k)
        times.append(t * cfg.N / n_rows)      # extrapolated full-matvec seconds
    sec = float(np.mean(times))
    val = 1.0 / sec
    line = {"metric": "gmres_matvecs_per_s", "value": val, "unit": "matvec/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{cfg.name} {args.mode}", "N": cfg.N, "eps": cfg.eps, "kind": cfg.kind,
                       "layout": cfg.layout, "tables": args.tables, "K": tab.K, "Kstar": tab.Kstar, "p": tab.p},
            "cpu_baseline": {"value": val, "unit": "matvec/s", "cores": thr, "kind": "oracle",
                             "sample": f"{n_rows} of {cfg.N} target patches per step, extrapolated x{cfg.N / n_rows:.1f}"},
            "e2e": {"value": val, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.mode is None:
        args.mode = "direct" if args.config in ("C1", "C2") else "hier"
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_1906_04209_b200 as nc
    from nc_inputs import CONFIGS, random_coeffs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus={args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    tab = make_tables(cfg, args.tables)
    centers = cfg.centers()
    mode = nc.NC_HIER if args.mode == "hier" else nc.NC_DIRECT
    nid = None
    if world > 1:
        obj = [nc.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    t_setup0 = time.perf_counter()
    h = nc.Handle(cfg.kind, centers, cfg.eps, tab, mode=mode, precision=cfg.precision, device=local, world=world,
                  rank=rank, nccl_id=nid)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup0
    x_all = random_coeffs(cfg.N, tab.K, 2000 + int(cfg.name[1:]))
    x = torch.from_numpy(h.to_internal(x_all)).cuda()
    y = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    flush = torch.empty(int(256 * 2**20 // 4), dtype=torch.float32, device="cuda")   # 256 MB > 126 MB L2

    for _ in range(max(args.warmup, 0)):
        h.matvec(x, y)
    torch.cuda.synchronize()

    # timed region: per-step CUDA events around each matvec on the launching stream, plus the library's own
    # events around the dominant kernel inside every timed matvec (nc_time_stages; no host sync inside nc_matvec)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stage_ms, launches = [], 0
    h.time_stages(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()                                   # L2 flush between timed steps (not timed)
            starts[k].record(stream)
            h.matvec(x, y)
            ends[k].record(stream)
            st = h.stats()                                  # waits for this step's stage events
            stage_ms.append(st["ms_last"][:8])
            launches += st["launches_per_matvec"]
        torch.cuda.synchronize()
    h.time_stages(False)
    if world > 1:
        dist.barrier()
    ms_steps = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms_total = float(np.sum(ms_steps))
    stages_avg = [float(v) for v in np.mean(np.asarray(stage_ms), axis=0)]
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    value = args.steps / (ms_total / 1e3)

    # end to end through the host-buffer C-ABI entry point (pinned host buffers, H2D + matvec + D2H)
    xh = torch.from_numpy(h.to_internal(x_all)).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    import ctypes
    from paper_1906_04209_b200.nc import _dp, _check
    h._L.nc_matvec_host(h._h, ctypes.cast(xh.data_ptr(), _dp), ctypes.cast(yh.data_ptr(), _dp))
    if world > 1:
        dist.barrier()
    n_e2e = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        _check(h._L.nc_matvec_host(h._h, ctypes.cast(xh.data_ptr(), _dp), ctypes.cast(yh.data_ptr(), _dp)))
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": n_e2e / e2e_s, "unit": "matvec/s", "steps": n_e2e, "h2d_bytes_per_step": int(xh.numel() * 8),
           "d2h_bytes_per_step": int(yh.numel() * 8)}

    # time to solution (GMRES from x0 = 0 on the physical right-hand side P.1, then the read-out)
    solve = None
    if not args.no_solve:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        h.time_stages(True)                 # events only (no host sync inside nc_matvec); GMRES CGS2 timing
        t0 = time.perf_counter()
        xs, its, hist = h.gmres(rtol=cfg.gmres_tol, max_iter=300, allow_noconv=True)
        Is, val = h.flux_or_mfpt(xs) if (cfg.kind == 1 or args.tables == "physical") else (float("nan"), float("nan"))
        tts = time.perf_counter() - t0
        h.time_stages(False)
        gst = h.stats()
        solve = {"time_to_solution_s": tts, "gmres_iters": its, "final_rel_residual": float(hist[-1]),
                 "I_sigma": Is, ("mu" if cfg.kind == 0 else "J"): val, "setup_s": setup_s,
                 "tables": args.tables}
        if gst["gmres_ortho_iters"] > 0 and gst["gmres_ortho_ms"] > 0:
            hbm = json.load(open(PEAKS_FILE)).get("hbm_gbs") if os.path.exists(PEAKS_FILE) else None
            gbs = gst["gmres_ortho_bytes"] / (gst["gmres_ortho_ms"] * 1e-3) / 1e9
            solve["gmres_cgs2"] = {"bound": "hbm", "ms_total": gst["gmres_ortho_ms"], "iters": gst["gmres_ortho_iters"],
                                   "achieved": gbs, "unit": "GB/s", "peak": hbm, "frac": gbs / hbm if hbm else None,
                                   "note": "CGS2 (2 x multidot + gemv_sub, norm): algorithmic bytes / device time; "
                                           "peak = MEASURED_PEAKS.json hbm_gbs (of measured)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    # roofline of the dominant kernel (direct: k_pairs_direct; hier: k_pairs_grid): FP64 pipe
    peaks = load_fp64_peak()
    pair_ms = stages_avg[2] if args.mode == "direct" else stages_avg[4]
    pairs = st["pairs_per_matvec"] if args.mode == "direct" else st["hier_grid_pairs"]
    kname = "k_pairs_direct" if args.mode == "direct" else "k_pairs_grid"
    fpp = st["pair_fp64_flops_direct"] if args.mode == "direct" else st["pair_fp64_flops_grid"]
    ipp = st["pair_fp64_inst_direct"] if args.mode == "direct" else st["pair_fp64_inst_grid"]
    roof = None
    if pair_ms > 0 and fpp:
        ach = pairs * fpp / (pair_ms * 1e-3) / 1e12
        peak = peaks.get("dfma")
        traffic, tsrc = profiled_traffic(kname, cfg.name, args.mode)
        roof = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": (ach / peak) if peak else None, "traffic": traffic,
                "fp64_flops_per_pair": fpp, "fp64_inst_per_pair": ipp,
                "fp64_pipe_util": (pairs * ipp / (pair_ms * 1e-3)) / (peak * 1e12 / 2) if peak else None,
                "kernel": kname, "kernel_ms": pair_ms, "kernel_share_of_step": pair_ms / (ms_total / args.steps),
                "note": "FP64 flops executed per pair by the running variant (SASS count, 2 per DFMA; nc_stats) x pairs "
                        "/ kernel ms (CUDA events around the kernel in every timed step); peak = measured DFMA "
                        "throughput (profiles/r02h_fp64_peak.txt, of measured, SM clock 1965 MHz under load); fp64_pipe_util = FP64 instructions / "
                        "(peak / 2); traffic = DRAM bytes per launch from " + (tsrc or "no capture"),
                "pairs_per_s": pairs / (pair_ms * 1e-3),
                "l1_shared_wavefront_bound": profiled_shared_wavefronts(kname, cfg.name, args.mode)}
    # the fp64 tensor-core GEMMs (K1 T-apply over the used rungs, K3 P-apply + identity): DMMA roofline
    kd = st["K"] * st["Kstar"] * 2.0 * st["row_count"]
    gemms = {}
    for name, ms, fl in (("T_apply", stages_avg[0], st["gemm_flops_per_matvec"] - kd), ("P_apply", stages_avg[3], kd)):
        if ms > 0:
            tf = fl / (ms * 1e-3) / 1e12
            gemms[name] = {"bound": "tensor", "kernel": "k_gemm_dmma", "ms": ms, "achieved": tf, "unit": "TFLOP/s",
                           "peak": peaks.get("dmma"), "frac": tf / peaks["dmma"] if peaks.get("dmma") else None}
    # issue-bound model of the dominant kernel: an FP64 warp instruction holds its SMSP's dispatch
    # 2 cycles, any other 1; per-pair counts from this build's SASS main loop (tools/sass_loop.py, cuobjdump)
    gv = st.get("grid_variant") or [0] * 8
    clk_hz = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
    if roof is not None:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            from sass_loop import main_loop
            import paper_1906_04209_b200 as ncmod
            # the variant in use (nc_stats grid_variant: nt, tpt, unroll, stage, far, tma, minb, persist)
            pat = (f"k_pairs_grid_wILi{cfg.kind}ELi{gv[1]}ELi{gv[2]}ELi{gv[4]}ELi{gv[0]}ELi{gv[6]}E"
                   if args.mode == "hier" else f"k_pairs_directILi{cfg.kind}ELi2ELb1E")
            ml = main_loop(ncmod.nc.LIB_PATH, pat)
            if ml:
                fp, oth = ml
                cyc = 2.0 * fp + oth
                ideal_ms = pairs / 32.0 * cyc / (148 * 4 * clk_hz) * 1e3
                roof["issue_model"] = {"fp64_inst_per_pair": fp, "other_inst_per_pair": oth,
                                       "cycles_per_warp_pair": cyc, "ideal_ms": ideal_ms,
                                       "frac": ideal_ms / pair_ms,
                                       "note": "2 dispatch cycles per FP64 warp instruction + 1 per other, SASS "
                                               "main loop of this build, 592 SMSPs at the sampled SM clock"}
        except Exception as e:  # pragma: no cover
            roof["issue_model"] = {"error": str(e)[:200]}
    # the same pair evaluation in isolation (sources in registers, no staging / barriers / partial warps), measured
    # in this run by nc_pair_mix on this GPU: the SMSP-cycles per warp-pair the hardware sustains for this loop body
    if roof is not None and args.mode == "hier" and gv[5] == 3:
        try:
            import paper_1906_04209_b200 as ncmod
            best = None
            for cps in (2, 3):
                ms_mix, wp = ncmod.pair_mix(cfg.kind, gv[4], cps)
                c_iso = ms_mix * 1e-3 * clk_hz * 148 * 4 / wp
                best = c_iso if best is None else min(best, c_iso)
            kc = pair_ms * 1e-3 * clk_hz * 148 * 4 / (pairs / 32.0)
            roof["instruction_mix_bound"] = {"cycles_per_warp_pair_isolated": best, "kernel_cycles_per_warp_pair": kc,
                                             "frac": best / kc,
                                             "source": "nc_pair_mix (libnc), measured in this run: best of 2-3 "
                                                       "CTAs/SM at the sampled SM clock"}
        except Exception as e:  # pragma: no cover
            roof["instruction_mix_bound"] = {"error": str(e)[:200]}
    # HBM-bound stages of the matvec (north_star: "HBM GB/s for the gather/scatter stages"): the grid reduction
    # (per-unit partial values in, grid values out) and the K1 outgoing GEMM with its scattered rho epilogue
    hbm_stages = None
    if args.mode == "hier" and len(stages_avg) > 7:
        hbm = json.load(open(PEAKS_FILE)).get("hbm_gbs") if os.path.exists(PEAKS_FILE) else None
        psum = (st["gemm_flops_per_matvec"] / (2.0 * st["row_count"]) - st["K"] * st["Kstar"]) / st["K"]
        red_b = 8.0 * (st["hier_unit_points"] + st["hier_grid_points"])
        k1_b = 8.0 * (st["N"] * st["K"] + psum * st["K"] + st["N"] * psum)
        hbm_stages = {}
        # the reduce stage's events bracket nothing when the reduction is fused into k_transform_w (R37): a real
        # k_reduce_chunks launch reads >= 1 GB at C5 and takes >= 0.2 ms, an empty bracket ~3 us
        fused = stages_avg[7] < 0.05
        for name, b, ms in (("k_reduce_chunks", red_b, None if fused else stages_avg[7]),
                            ("K1_T_apply_scatter", k1_b, stages_avg[0])):
            if ms:
                gbs = b / (ms * 1e-3) / 1e9
                hbm_stages[name] = {"bytes": b, "ms": ms, "achieved": gbs, "unit": "GB/s", "peak": hbm,
                                    "frac": gbs / hbm if hbm else None}
        if fused:
            hbm_stages["grid_reduce"] = ("fused into k_transform_w (R37): each warp sums its grid's partial values "
                                         "straight into shared memory; %.3g GB of partials read per matvec, timed "
                                         "inside hier_rest" % (8.0 * st["hier_unit_points"] / 1e9))
        hbm_stages["note"] = ("algorithmic bytes: the grid reduction reads every work unit's partial values and writes "
                              "the grid values; K1 reads X and the rungs' T and writes rho compactly (8 B per value); "
                              "peak = MEASURED_PEAKS.json hbm_gbs")
    # NEXT-3: the field of the solution on the sphere of radius 1 -+ eps/5, where the paper plots the MFPT (PAPER.md:2069-2097,
    # Fig. sphereplots): nc_field_near (host points in, values and v-bar out, synchronous; the patches within 4 eps of a
    # point from their density, the others from their compressed skeleton), Fibonacci points
    field = None
    if world == 1 and solve is not None and getattr(tab, "near_sigma", None) is not None and args.field_points > 0:
        n_f = args.field_points
        k = np.arange(n_f) + 0.5
        zf = 1.0 - 2.0 * k / n_f
        phi = np.pi * (1.0 + 5.0 ** 0.5) * k
        rf = 1.0 - cfg.eps / 5 if cfg.kind == 0 else 1.0 + cfg.eps / 5
        pts = rf * np.stack([np.sqrt(1 - zf * zf) * np.cos(phi), np.sqrt(1 - zf * zf) * np.sin(phi), zf], 1)
        want_mfpt = cfg.kind == 0 and args.tables == "physical"
        h.field_near(xs, pts[:8], tab, mfpt=want_mfpt)   # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        vf, mf, nnear = h.field_near(xs, pts, tab, mfpt=want_mfpt)
        tf = time.perf_counter() - t0
        fpairs = float(n_f) * cfg.N * tab.p
        field = {"points": n_f, "radius": rf, "near_pairs": nnear, "far_pairs": fpairs, "ms": tf * 1e3,
                 "points_per_s": n_f / tf, "mean_value": float(np.mean(vf)),
                 "note": "nc_field_near end to end (H2D points, compressed field of every patch, near pairs, density "
                         "quadrature of the near patches, D2H values)"}
        if want_mfpt:
            field.update({"mfpt_mean": float(np.mean(mf)), "mfpt_min": float(np.min(mf)), "mfpt_max": float(np.max(mf))})
            v0, m0, _ = h.field_near(xs, np.zeros((1, 3)), tab, mfpt=True)
            field["v_origin"], field["mfpt_origin"] = float(v0[0]), float(m0[0])
    # NEXT-4: the paper's accuracy metric eq:l2res (relative L2 residual of the multiple-scattering system on a
    # patch, on the tables' independent residual grid) for 16 seeded random patches of the solved system
    residual = None
    if world == 1 and solve is not None and getattr(tab, "res_S", None) is not None:
        pats = np.random.default_rng(77).choice(cfg.N, min(16, cfg.N), replace=False)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rv, _ = h.residual(xs, pats, tab)
        residual = {"patches": int(len(pats)), "max": float(np.max(rv)), "median": float(np.median(rv)),
                    "ms": (time.perf_counter() - t0) * 1e3, "grid_points": int(tab.res_w.size),
                    "note": "eq:l2res on 16 seeded random patches (nc_residual); the one-patch tables' own residual "
                            "(eq:patcherrl2) at this eps bounds it from below"}
    # the other BASELINE config with a direct mode, measured in the same run (secondary; not the headline metric):
    # C2 (exterior, N = 1000) direct, physical tables, 3 warm-up + 5 timed matvecs with CUDA events
    secondary = None
    if world == 1 and solve is not None and args.config == "C5":
        cfg2 = CONFIGS["C2"]
        tab2 = make_tables(cfg2, args.tables)
        h2 = nc.Handle(cfg2.kind, cfg2.centers(), cfg2.eps, tab2, mode=nc.NC_DIRECT)
        x2 = torch.from_numpy(h2.to_internal(random_coeffs(cfg2.N, tab2.K, 2002))).cuda()
        y2 = torch.empty_like(x2)
        for _ in range(3):
            h2.matvec(x2, y2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            h2.matvec(x2, y2)
        e1.record(stream)
        torch.cuda.synchronize()
        ms2 = e0.elapsed_time(e1) / 5
        st2 = h2.stats()
        secondary = {"workload": "C2 direct", "value": 1e3 / ms2, "unit": "matvec/s", "ms_per_matvec": ms2,
                     "pairs_per_matvec": st2["pairs_per_matvec"],
                     "pairs_per_s": st2["pairs_per_matvec"] / (ms2 * 1e-3),
                     "note": "whole matvec (K1 + pair sums + K3); most pairs take the far form (DESIGN.md R30: "
                             "15 FP64 instructions, exact form 19)"}
        h2.close()
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            # >= 16 sampled target patches; small configs calibrate to ~12 s of CPU work
            n_rows = args.cpu_sample or (max(16, auto_sample_rows(cfg, tab)) if cfg.N <= 10000 else 16)
            t, rows, thr = cpu_oracle_sample(cfg, tab, x_all, n_rows)
            cpu = {"value": 1.0 / (t * cfg.N / n_rows), "unit": "matvec/s", "cores": thr, "kind": "oracle",
                   "sample": f"{n_rows} of {cfg.N} target patches (direct sum), extrapolated x{cfg.N / n_rows:.1f}"}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "error": str(e)}
    line = {"metric": "gmres_matvecs_per_s", "value": value, "unit": "matvec/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{cfg.name} {args.mode}", "N": cfg.N, "eps": cfg.eps, "kind": cfg.kind,
                       "layout": cfg.layout, "tables": args.tables, "K": tab.K, "Kstar": tab.Kstar, "p": tab.p},
            "l2": "flushed between timed steps (256 MB write, untimed)",
            "clocks": clk.summary(), "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roof, "gemm_roofline": gemms, "cpu_baseline": cpu,
            "stages_ms": dict(zip(["T_apply", "all_gather", "direct_pairs", "P_apply", "grid_pairs", "hier_rest",
                                   "total", "grid_reduce"], stages_avg)), "pairs_per_matvec": st["pairs_per_matvec"],
            "hbm_stages": hbm_stages,
            "hier": ({k: st[k] for k in ("tree_levels", "tree_groups", "hier_grid_pairs", "hier_near_pairs",
                                         "hier_interp_terms", "hier_grid_points", "hier_grid_units", "hier_grid_fill",
                                         "hier_grid_warp_fill")}
                     if args.mode == "hier" else None),
            "solve": solve, "field": field, "residual": residual, "secondary": secondary}
    print(json.dumps(line), flush=True)
    h.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

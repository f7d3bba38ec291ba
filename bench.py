#!/usr/bin/env python
"""Benchmark: full branch-length-gradient evaluations per second (BJ:metric).

One step = one full evaluation of the hot path:
transition matrices from the eigensystem for new branch lengths, post-order
pruning, root likelihood, pre-order partials, per-edge gradient, the pattern
reduction and -- at N > 1 GPUs -- the NCCL allreduce of [logL, g].

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--precision fp64]
    torchrun --nproc-per-node N bench.py --gpus N ...      (patterns sharded, strong scaling)
    python bench.py --impl reference ...                    (the CPU oracle as the reference arm)

Timing: K device-timed steps (CUDA events on the instance stream), L2 flushed
between timed steps (outside the events), barrier + synchronize on both
sides, max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import phylo_synth as ps  # noqa: E402

METRIC = "full BLS-gradient evals/sec"
UNIT = "evals/s"
CONFIG_NAMES = {0: "jc5_c200", 1: "dengue997_hky_g4_c10000", 2: "carnivore62_mmm16_c5000",
                3: "yeast49_gy94_g4_c4000", 4: "wnv104_gy94_g4_ucld_c3700",
                5: "yeast49_mmm2x61_c4000", 6: "codonmmm4x61_10001_c256"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between timed steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra-configs", action="store_true",
                    help="skip the codon / MMM workloads timed beside the default dengue line")
    ap.add_argument("--no-fp64-probe", action="store_true", help="skip the in-run FP64 peak measurement")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the baseline sample")
    ap.add_argument("--virtual-shard", type=int, default=0, metavar="G",
                    help="evidence runs only: time rank 0's pattern shard of a G-GPU run on this one GPU "
                         "(value = that shard's evals/s; not a bench line)")
    ap.add_argument("--patterns", type=int, default=0, metavar="C",
                    help="evidence runs only (pattern-count sweep, SURVEY §8(f) NEXT-3): the config's "
                         "workload with C unique patterns instead of its default; not a bench line")
    return ap.parse_args()


def workload_name(cfg: int, C: int) -> str:
    base = CONFIG_NAMES[cfg]
    return base if cfg == 0 else base[:base.rfind("_c")] + f"_c{C}"


def make_problem(cfg: int, precision: str, patterns: int = 0):
    kw = {"precision": precision} if cfg in (1, 2, 3, 4, 5, 6) else {}
    if patterns > 0:
        kw["C"] = patterns
    return ps.make_config(cfg, **kw)


def dtype_name(precision: str) -> str:
    return "f64" if precision == "fp64" else "f32"


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------- roofline ----

def padded_states(S: int) -> int:
    return 4 if S <= 4 else 8 if S <= 8 else 16 if S <= 16 else 32 if S <= 32 else 64 if S <= 64 else 128 if S <= 128 else 256


def hbm_counts(pb, C: int, precision: str) -> dict:
    """Byte counts of one evaluation over C patterns; V = R C Sp w
    is one node's partials.
      b_min     5 (N-2) V + tips + 8 (N-1) C: the roofline basis (u written once
                and read twice, q written and read once, tip codes read twice,
                int32 scale exponents written and read); tips = 2 N C (int8
                codes) or 2 N C Sp w (partial tips, MMM);
      schedule  what this build's one-launch walk must move: 2 (N-2) V (u
                written once, read once; q never leaves the chip) + tips + 8 C;
      paper     (10N - 13) V, the paper-literal per-node schedule."""
    N, S, R = pb.n_tips, pb.states, len(pb.cat_rates)
    Sp = padded_states(S)
    w = 8 if precision == "fp64" else 4
    V = R * C * Sp * w
    tips = 2 * N * C if not pb.has_partials else 2 * N * C * Sp * w
    return {"b_min": 5 * (N - 2) * V + tips + 8 * (N - 1) * C,
            "schedule": 2 * (N - 2) * V + tips + 8 * C,
            "paper": (10 * N - 13) * V}


def flop_counts(pb, C: int) -> dict:
    """f_min = 3 (N-2) 2 S^2 R C (unpadded S); paper-literal
    (6N - 8) 2 Sp^2 R C."""
    N, S, R = pb.n_tips, pb.states, len(pb.cat_rates)
    Sp = 64 if S <= 64 else 128 if S <= 128 else 256
    return {"f_min": 3 * (N - 2) * 2 * S * S * R * C, "paper": (6 * N - 8) * 2 * Sp * Sp * R * C}


def tf32_peak(peaks):
    """Dense TF32 tensor peak: the measured bf16 burst peak x the guide's
    nominal tf32 / bf16 ratio (1.1 / 2.25 PFLOP/s, B200_PROFILING.md)."""
    return peaks.get("bf16_tflops", 1590.0) * 1.1 / 2.25


def load_peaks():
    """HBM: MEASURED_PEAKS.json (driver-written copy bandwidth).  FP64: measured
    inside this bench run (probe_fp64, below) when it ran, else our committed
    microbenchmark (profiles/r01/fp64_peak.json)."""
    out = {}
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        out.update(hbm_gbs=float(d["hbm_gbs"]), hbm_src="measured (MEASURED_PEAKS.json hbm_gbs)",
                   bf16_tflops=float(d["bf16_tflops"]))
    except Exception:
        out.update(hbm_gbs=6650.0, hbm_src="fallback (B200_PROFILING.md)", bf16_tflops=1590.0)
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01", "fp64_peak.json")))
        out.update(fp64_tflops=float(d["dmma_tflops"]), dfma_tflops=float(d["dfma_tflops"]),
                   fp64_src="committed DMMA microbenchmark (profiles/r01/fp64_peak.json)",
                   dfma_src="committed DFMA microbenchmark (profiles/r01/fp64_peak.json)")
    except Exception:
        out.update(fp64_tflops=37.0, dfma_tflops=36.0, fp64_src="fallback (~37 TF/s)", dfma_src="fallback")
    # FP32 FFMA: 148 SMs x 128 lanes x 2 flops x 1.965 GHz (guide unit counts, max clock)
    out.update(ffma_tflops=148 * 128 * 2 * 1.965e9 / 1e12, ffma_src="derived: 148 SMs x 128 FP32 lanes x 2 x 1.965 GHz")
    return out


def probe_fp64(peaks, device: int):
    """FP64 DMMA / DFMA peaks measured now, on this GPU, with clocks sampled
    during the probe (lib/libpgprobe.so, csrc/probe.cu)."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2303_04390_b200", "lib", "libpgprobe.so"))
    dm, df, n = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int(0)
    with ClockSampler(device) as clk:
        rc = lib.pgprobe_fp64_peak(int(device), ctypes.c_float(1500.0), ctypes.byref(dm), ctypes.byref(df),
                                   ctypes.byref(n))
    if rc != 0:
        return {"error": f"probe rc {rc}"}
    peaks.update(fp64_tflops=dm.value, dfma_tflops=df.value,
                 fp64_src="measured in this run (mma.sync m8n8k4 f64 DMMA probe, csrc/probe.cu)",
                 dfma_src="measured in this run (DFMA probe, csrc/probe.cu)")
    return {"dmma_tflops": round(dm.value, 3), "dfma_tflops": round(df.value, 3), "launches": n.value,
            "how": "best launch of 592 CTAs x 8 warps, ~1.5 s per probe", "clocks": clk.summary()}


def traffic_key(cfg: int, precision: str, shard: int = 1, patterns: int = 0) -> str:
    k = f"config{cfg}_{precision}"
    if shard > 1:
        k += f"_shard{shard}"
    if patterns > 0:
        k += f"_C{patterns}"
    return k


def load_traffic(key: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from a
    committed ncu --set full capture of exactly this workload
    (profiles/ncu_traffic.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(key)
        return None if d is None else d["bytes"]
    except Exception:
        return None


def roofline(pb, C: int, variant: int, precision: str, kms: dict, peaks: dict, traffic, flow: bool,
             eval_ms: float) -> dict:
    """Roofline object of the dominant kernel (the traversal) on SURVEY §8(d)'s
    algorithmic basis: B_min for the HBM-bound S <= 16 paths, F_min for the
    FP64 tensor path; the schedule / paper-literal / ncu-DRAM figures beside.
    kernel_ms is the traversal's event-timed duration (separate timing pass);
    eval_frac uses the whole measured evaluation (A1 + traversal + reduction,
    as timed per step)."""
    t = kms["traverse"] * 1e-3
    ev = eval_ms * 1e-3
    if variant in (1, 2, 3, 4):
        fl = flop_counts(pb, C)
        hb = hbm_counts(pb, C, precision)
        if variant == 4:
            pk, unit, bound = tf32_peak(peaks), "TFLOP/s", "tensor"
            src = ("dense TF32 = measured bf16 burst peak (MEASURED_PEAKS.json) x nominal 1.1/2.25; "
                   "each product issues 3 TF32 MMAs (3xTF32), so 1/3 of this is the fp32-accurate ceiling")
            kname = "tc_post_kernel + tc_pre_kernel (tcgen05 kind::tf32, 3xTF32, all levels)"
        elif variant >= 2:
            pk, unit, bound, src = peaks["fp64_tflops"], "TFLOP/s", "tensor", peaks["fp64_src"]
            kname = ("big_post_kernel + big_pre_kernel (S = 256 class, transpose-free, all levels)" if variant == 3
                     else "codon_flow2_kernel (post + pre order, one launch, TMA ring)" if flow
                     else "codon_post_kernel + codon_pre_kernel (all levels of one evaluation)")
        else:
            pk, src = ((peaks["dfma_tflops"], peaks["dfma_src"]) if precision == "fp64"
                       else (peaks["ffma_tflops"], peaks["ffma_src"]))
            unit, bound, kname = "TFLOP/s", "alu", "traverse_large_kernel (SIMT)"
        ach = fl["f_min"] / t / 1e12
        r = {"bound": bound, "achieved": round(ach, 3), "peak": round(pk, 3), "unit": unit,
             "frac": round(ach / pk, 4), "traffic": traffic, "kernel": kname,
             "basis": "SURVEY §8(d) F_min = 3(N-2) 2 S^2 R C (unpadded S) per launch",
             "algorithmic_flops_per_launch": fl["f_min"], "kernel_ms": round(kms["traverse"], 5),
             "eval_ms": round(ev * 1e3, 5), "eval_frac": round(fl["f_min"] / ev / 1e12 / pk, 4),
             "paper_literal": {"flops": fl["paper"], "frac": round(fl["paper"] / t / 1e12 / pk, 4)},
             "peak_source": src}
        if traffic:
            r["dram_frac_ncu"] = round(traffic / t / 1e9 / peaks["hbm_gbs"], 4)
            r["hbm_b_min_frac"] = round(hb["b_min"] / t / 1e9 / peaks["hbm_gbs"], 4)
        return r
    hb = hbm_counts(pb, C, precision)
    ach = hb["b_min"] / t / 1e9
    pk = peaks["hbm_gbs"]
    r = {"bound": "hbm", "achieved": round(ach, 1), "peak": pk, "unit": "GB/s", "frac": round(ach / pk, 4),
         "traffic": traffic, "kernel": "traverse_small_kernel",
         "basis": "SURVEY §8(d) B_min = 5(N-2)V + 2NC + 8(N-1)C, V = R C Sp w (per launch)",
         "algorithmic_bytes_per_launch": hb["b_min"], "kernel_ms": round(kms["traverse"], 5),
         "eval_ms": round(ev * 1e3, 5), "eval_frac": round(hb["b_min"] / ev / 1e9 / pk, 4),
         "schedule_bytes_per_launch": hb["schedule"],
         "schedule_frac": round(hb["schedule"] / t / 1e9 / pk, 4),
         "paper_literal": {"bytes": hb["paper"], "frac": round(hb["paper"] / t / 1e9 / pk, 4)},
         "peak_source": peaks["hbm_src"]}
    if traffic:
        r["dram_frac_ncu"] = round(traffic / t / 1e9 / pk, 4)
    return r


def pct(xs, q):
    return float(np.percentile(np.asarray(xs), q))


# ------------------------------------------------------------ CPU oracle ----

def cpu_oracle_rate(pb, seconds: float, threads: int):
    """Oracle evals/s on a bounded pattern sample with `threads` host threads
    (pattern blocks run concurrently, the paper's CPU parallelisation P:78)."""
    import oracle
    C = pb.patterns
    m0 = min(C, max(threads * 4, 16))
    t0 = time.perf_counter()
    oracle.loglik_grad(pb, 0, m0, threads=threads, block=max(1, m0 // threads))
    dt0 = time.perf_counter() - t0
    m = int(min(C, max(m0, m0 * seconds / max(dt0, 1e-6))))
    reps, dt = 0, 0.0
    while reps == 0 or (dt < 0.5 * seconds and reps < 50):     # whole workload faster than the budget: repeat
        t0 = time.perf_counter()
        oracle.loglik_grad(pb, 0, m, threads=threads, block=max(1, -(-m // (threads * 4))))
        dt += time.perf_counter() - t0
        reps += 1
    rate = reps * (m / C) / dt
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"patterns [0,{m}) of {C} (full tree) x {reps} evaluation(s), {dt:.1f} s, scaled by C/{m}"}


def workload_config(args, pb, C, world, lo=0, hi=None, flushed=True, shard=0):
    """The `config` object (identical in both arms)."""
    return {"workload": workload_name(args.config, C), "tips": pb.n_tips, "patterns": C,
            "states": pb.states, "categories": len(pb.cat_rates), "precision": args.precision,
            "l2": "flushed (256 MiB write) between timed steps" if flushed else "not flushed",
            "parallelism": (f"pattern-shard x{world}" if shard <= 1 else
                            f"virtual: rank 0's shard [{lo},{hi}) of x{shard}, on 1 GPU"),
            "branch_lengths": "seeded +-1% jitter per step"}


# ------------------------------------------------------------------ ours ----

def time_steps(step, stream, steps, warmup, flush, inst=None, ksteps=32):
    """Warm-up, then `steps` steps each bracketed by CUDA events on `stream`
    (L2 flushed outside the events).  Then, separately, `ksteps` more steps
    with the instance's in-graph kernel events enabled give the per-kernel
    split (events between kernels also switch off the A1 -> flow
    programmatic launch, so the split is not taken from the timed steps)."""
    import torch
    kt = {"pmat": 0.0, "traverse": 0.0, "reduce": 0.0}
    with torch.cuda.stream(stream):
        for i in range(warmup):
            step(i)
        stream.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            if flush is not None:
                flush.zero_()
            evs[k][0].record(stream)
            step(warmup + k)
            evs[k][1].record(stream)
        stream.synchronize()
        if inst is not None and ksteps > 0:
            inst.set_kernel_timing(True)
            for k in range(ksteps + 2):
                if flush is not None:
                    flush.zero_()
                step(warmup + k % max(steps, 1))
                if k >= 2:
                    t = inst.kernel_times()
                    for n in kt:
                        kt[n] += t[n] / ksteps
            inst.set_kernel_timing(False)
            stream.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    return ms, kt


def bench_instance(pb, precision, device, lo, hi, steps, warmup, flush, seed_off=99):
    """Single-process timing of one (shard of a) workload; returns stats."""
    import torch
    import paper_2303_04390_b200 as pg
    dev = torch.device("cuda", device)
    inst = pg.from_problem(pb, precision=precision, device=device, lo=lo, hi=hi)
    B = 2 * pb.n_tips - 2
    out = torch.zeros(B + 1, dtype=torch.float64, device=dev)
    rng = np.random.default_rng(ps.MASTER_SEED + seed_off)
    bls = pb.branch_lengths[None, :] * rng.uniform(0.99, 1.01, size=(warmup + steps, B))
    bl_dev = torch.tensor(bls, dtype=torch.float64, device=dev)

    def step(i):
        inst.set_branch_lengths_device(bl_dev[i])
        inst.compute_device(out)

    ms, kt = time_steps(step, inst.stream, steps, warmup, flush, inst)
    zp = inst.check_status()
    assert zp < 0, f"zero likelihood at pattern {zp}"
    info = inst.plan_info()
    nk = inst.kernels_per_eval()
    return inst, ms, kt, info, nk, bls


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2303_04390_b200 as pg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    peaks = load_peaks()
    fp64_probe = None
    if rank == 0 and world == 1 and not args.no_fp64_probe:
        fp64_probe = probe_fp64(peaks, local)

    pb = make_problem(args.config, args.precision, args.patterns)
    C = pb.patterns
    B = 2 * pb.n_tips - 2
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    shard = args.virtual_shard if args.virtual_shard > 1 else 0
    if shard:
        assert world == 1, "--virtual-shard is a single-process emulation"
        lo, hi = pg.shard_range(C, shard, 0)
    else:
        lo, hi = pg.shard_range(C, world, rank)

    rng = np.random.default_rng(ps.MASTER_SEED + 99)
    nvar = args.warmup + args.steps
    bls = pb.branch_lengths[None, :] * rng.uniform(0.99, 1.01, size=(nvar, B))
    bl_dev = torch.tensor(bls, dtype=torch.float64, device=dev)

    # one CUDA graph per step: [branch lengths D2D, evaluation kernels, allreduce]
    # at N > 1 (the library enqueues into the caller's capture)
    ev = pg.ShardEvaluation(pb, rank=0 if shard else rank, world=shard or world, device=local,
                            precision=args.precision, capture=world > 1, timing=world > 1)
    inst = ev.inst

    def step(i):
        with torch.cuda.stream(ev.stream):
            ev.bl.copy_(bl_dev[i], non_blocking=True)
        ev.evaluate()

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms, kt = time_steps(step, ev.stream, args.steps, args.warmup, flush, inst)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    zp = ev.zero_pattern()
    assert zp < 0, f"zero likelihood at pattern {zp}"
    dev_ms = sum(ms)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    value = 1000.0 / ms_per_step            # whole-job evaluations per second

    # ---- end to end through the public API with host buffers ---------------
    e2e_steps = max(10, min(args.steps, 200))
    host_out = torch.empty(B + 1, dtype=torch.float64, pin_memory=True)
    host_bl = torch.empty(B, dtype=torch.float64, pin_memory=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        if world == 1 and inst is not None:
            inst.set_branch_lengths(bls[k % nvar])           # pg_set_branch_lengths (pinned staging)
            logl, g = inst.compute()                           # pg_compute: H2D, graph, D2H, sync
        else:
            host_bl.copy_(torch.from_numpy(bls[k % nvar]))
            with torch.cuda.stream(ev.stream):
                ev.bl.copy_(host_bl, non_blocking=True)
                ev.evaluate()
                host_out.copy_(ev.out, non_blocking=True)
            ev.stream.synchronize()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_rate = e2e_steps / float(te.item())

    result = None
    if rank == 0:
        info = inst.plan_info() if inst is not None else {}
        nk = inst.kernels_per_eval() if inst is not None else 0
        variant = info.get("kernel_variant", 0)
        Cl = hi - lo
        traffic = load_traffic(traffic_key(args.config, args.precision, shard, args.patterns))
        result = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "ms_step_p10_p50_p90": [round(pct(ms, 10), 5), round(pct(ms, 50), 5), round(pct(ms, 90), 5)],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype_name(args.precision), "data": "synthetic",
            "config": workload_config(args, pb, C, world, lo, hi, flush is not None, shard),
            "e2e": {"value": round(e2e_rate, 3), "unit": UNIT, "h2d_bytes_per_step": 8 * B,
                    "d2h_bytes_per_step": 8 * (B + 1) + (4 if world == 1 else 0),
                    "path": ("pg_set_branch_lengths + pg_compute (host buffers)" if world == 1 else
                             "pinned H2D of b, captured [b, evaluation, NCCL allreduce] graph, D2H of [logL, g]")},
            "gpu_launches": args.steps * nk,
            "roofline": roofline(pb, Cl, variant, args.precision, kt, peaks, traffic, info.get("flow_tiles", 0) > 0,
                                 ms_per_step),
            "kernel_ms": {k: round(v, 5) for k, v in kt.items()},
            "kernel_ms_note": "per-kernel split from a separate 32-step pass with in-graph events (A1 -> flow PDL off)",
            "plan": info,
            "clocks": clk.summary(),
        }
        if world > 1:
            result["allreduce"] = "NCCL allreduce of 2N-1 doubles captured in the per-step CUDA graph"
        if fp64_probe is not None:
            result["fp64_peak_probe"] = fp64_probe
    ev.close()
    return result, pb


def run_extra_configs(args, peaks):
    """The codon (FP64 tensor) workloads beside the headline line, each timed
    on this GPU with the same protocol (BJ:configs[3], [4], and rank 0's
    shard of the 8-GPU yeast and WNV runs -- BJ:configs[4] is the sharded
    workload)."""
    import torch
    dev = torch.device("cuda", 0)
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    out = {}
    steps, warmup = min(args.steps, 200), max(3, min(args.warmup, 20))
    import paper_2303_04390_b200 as pg
    for cfg, shard in ((3, 0), (4, 0), (3, 8), (4, 8), (2, 0), (5, 0)):
        pb = make_problem(cfg, "fp64")
        C = pb.patterns
        lo, hi = pg.shard_range(C, shard, 0) if shard else (0, C)
        inst, ms, kt, info, nk, _ = bench_instance(pb, "fp64", 0, lo, hi, steps, warmup, flush, 100 + cfg)
        inst.close()
        name = workload_name(cfg, C) + (f"_shard0of{shard}" if shard else "")
        mps = sum(ms) / len(ms)
        out[name] = {"value": round(1000.0 / mps, 3), "unit": UNIT, "ms_per_step": round(mps, 5),
                     "ms_step_p10_p50_p90": [round(pct(ms, 10), 5), round(pct(ms, 50), 5), round(pct(ms, 90), 5)],
                     "patterns_timed": hi - lo, "steps": steps, "warmup": warmup,
                     "kernel_ms": {k: round(v, 5) for k, v in kt.items()},
                     "roofline": roofline(pb, hi - lo, info["kernel_variant"], "fp64", kt, peaks,
                                          load_traffic(traffic_key(cfg, "fp64", shard)), info.get("flow_tiles", 0) > 0,
                                          mps),
                     "plan": info}
        if shard:
            out[name]["note"] = (f"one GPU timing rank 0's pattern shard [{lo},{hi}) of a {shard}-GPU run "
                                 "(the per-GPU work of that run; the allreduce of 2N-1 doubles is not included)")
    return out

def run_reference(args):
    """The CPU oracle as the reference arm (this tier has no installable
    reference: /root/reference holds only the paper), on our arm's config,
    metric and unit; rank 0 alone runs it."""
    import oracle
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    pb = make_problem(args.config, args.precision, args.patterns)
    C = pb.patterns
    threads = os.cpu_count() or 1
    # size the per-step sample so the whole run takes ~2-3 minutes
    m0 = min(C, threads * 4)
    t0 = time.perf_counter()
    oracle.loglik_grad(pb, 0, m0, threads=threads, block=max(1, m0 // threads))
    per_pat = (time.perf_counter() - t0) / m0
    budget = 150.0 / max(1, args.steps + min(args.warmup, 3))
    m = int(max(threads, min(C, budget / per_pat)))
    for _ in range(min(args.warmup, 3)):
        oracle.loglik_grad(pb, 0, m, threads=threads, block=max(1, -(-m // threads)))
    times = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        oracle.loglik_grad(pb, 0, m, threads=threads, block=max(1, -(-m // threads)))
        times.append(time.perf_counter() - t0)
    step_s = sum(times) / len(times)
    value = (m / C) / step_s
    sample = f"patterns [0,{m}) of {C} per step (full tree), scaled by C/{m}"
    cfg = workload_config(args, pb, C, world, flushed=not args.no_flush)   # identical to our arm's
    return {"impl": "reference", "note": "host CPU oracle: config.l2 describes the GPU arm's timing", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1000.0 / value, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": threads,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res, pb = run_ours(args)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank == 0:
        if world == 1 and not args.no_extra_configs and args.config == 1 and args.patterns == 0 \
                and args.virtual_shard <= 1:
            peaks = load_peaks()
            if "fp64_peak_probe" in res and "dmma_tflops" in res["fp64_peak_probe"]:
                peaks.update(fp64_tflops=res["fp64_peak_probe"]["dmma_tflops"],
                             dfma_tflops=res["fp64_peak_probe"]["dfma_tflops"],
                             fp64_src="measured in this run (DMMA probe, csrc/probe.cu)",
                             dfma_src="measured in this run (DFMA probe, csrc/probe.cu)")
            res["configs"] = run_extra_configs(args, peaks)
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_oracle_rate(pb, args.cpu_seconds, os.cpu_count() or 1)
            res["cpu_baseline_1thread"] = cpu_oracle_rate(pb, args.cpu_seconds / 2, 1)
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Benchmark: NSGA-III on LSMOP1 (m=3, d=1000, pop 200k) -- generations/sec on B200.

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl reference]
One JSON line on rank 0.  A step is one full NSGA-III generation (pair ->
SBX -> PM -> LSMOP1 evaluation -> shuffle -> ND sort -> normalize ->
associate -> niche fill -> survivor gather) of the north-star workload
(BASELINE.json configs[3] at pop 200k, the north-star target), population
resident in HBM.  ``value`` is whole-job gens/s; ``e2e`` is the same loop
through the public harness API with the per-step host inputs (the host RNG's
permutations) uploaded from pinned memory and the new objective matrix read
back every step.  ``--impl reference`` times the CPU oracle port of the
reference on bounded samples on the host cores.
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
sys.path.insert(0, ROOT)

METRIC = "generations/sec (NSGA-III, LSMOP1 m=3 d=1000)"
UNIT = "gen/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pop", type=int, default=200_000)
    ap.add_argument("--dim", type=int, default=1000)
    ap.add_argument("--objectives", type=int, default=3)
    ap.add_argument("--problem", default="lsmop1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-pop", type=int, default=4000)
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------- CPU baseline
def cpu_sample(pop, dim, m, problem, seed=0, reps=1):
    """Seconds per oracle generation at population ``pop`` (the reference algorithm on the host)."""
    from oracle import directions as odir
    from oracle import generation, problems as oprob

    if problem == "lsmop1":
        dim = oprob.lsmop_dimension(m, dim)  # PlatEMO's D for the requested dimension
        lower, upper = oprob.lsmop_bounds(m, dim)
    else:
        lower, upper = np.zeros(dim), np.ones(dim)
    W = odir.simplex_lattice(m, odir.largest_h_for(pop, m))
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
    X = lower + rng.random((pop, dim)) * (upper - lower)
    F = oprob.evaluate(problem, X, m)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        X, F = generation.nsga3_generation(X, F, W, pop, rng, problem, m, lower, upper)
        times.append(time.perf_counter() - t0)
    return min(times)


def cpu_baseline(args):
    """Oracle port timed on a bounded sample, extrapolated (N^2) to the workload's pop."""
    small = max(args.cpu_sample_pop // 2, 100)
    t_small = cpu_sample(small, args.dim, args.objectives, args.problem)
    t_big = cpu_sample(args.cpu_sample_pop, args.dim, args.objectives, args.problem)
    expo = float(np.log(t_big / t_small) / np.log(args.cpu_sample_pop / small))
    scale = (args.pop / args.cpu_sample_pop) ** 2  # conservative: measured exponent is >= 2
    t_full = t_big * scale
    return {
        "value": 1.0 / t_full,
        "unit": UNIT,
        "cores": os.cpu_count(),
        "kind": "port",
        "sample": (f"oracle (NumPy restatement of temo) full NSGA-III generation at pop "
                   f"{args.cpu_sample_pop} ({t_big:.3f} s) and {small} ({t_small:.3f} s, local "
                   f"exponent {expo:.2f}); value extrapolated by (pop ratio)^2 to pop {args.pop}; "
                   f"NumPy ufuncs single-threaded, OpenBLAS threads={os.environ.get('OPENBLAS_NUM_THREADS', 'all')}"),
        "measured_s_per_gen_at_sample": t_big,
    }


def reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    steps = []
    for _ in range(args.warmup):
        cpu_sample(args.cpu_sample_pop, args.dim, args.objectives, args.problem)
    for s in range(args.steps):
        steps.append(cpu_sample(args.cpu_sample_pop, args.dim, args.objectives, args.problem, seed=s))
    t = statistics.mean(steps) * (args.pop / args.cpu_sample_pop) ** 2
    v = 1.0 / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": f"each step: one oracle NSGA-III generation at pop {args.cpu_sample_pop}, "
                                   f"extrapolated by (pop ratio)^2 to pop {args.pop}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args):
    N = 2 * args.pop
    return {"workload": f"NSGA-III {args.problem.upper()} m={args.objectives} d={args.dim} pop={args.pop} "
                        f"(merged N={N}); BASELINE.json configs[3] at the north-star size",
            "pop": args.pop, "merged_N": N, "dim": args.dim, "objectives": args.objectives,
            "problem": args.problem, "rng": "NumPy Philox stream (host permutations, device uniforms)",
            "l2": "inputs larger than L2 (X 3.2 GB merged, dominance bitmap 10 GB)",
            "parallelism": (f"ND sort column-sharded over {args.gpus} GPUs (NCCL all-gather of the N-bit front "
                            f"mask per front), other stages replicated" if args.gpus > 1 else "single GPU")}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index=0):
        self.proc = None
        self.lines = []
        self.index = index

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- roofline
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback (no MEASURED_PEAKS.json)


def hbm_peak():
    """(GB/s, source) from the driver-written MEASURED_PEAKS.json, else the recipe's fallback."""
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for key in ("hbm_gbs", "hbm_GBps", "hbm_copy_gbs"):
            if key in peaks:
                return float(peaks[key]), f"of measured (MEASURED_PEAKS.json {key})"
        for key, v in peaks.items():
            if "hbm" in key.lower() and isinstance(v, (int, float)):
                return float(v), f"of measured (MEASURED_PEAKS.json {key})"
    except Exception:
        pass
    return FALLBACK_HBM_GBS, "of fallback (B200_PROFILING.md: 6.65 TB/s; MEASURED_PEAKS.json absent)"


def k1_bytes(N, ws=1):
    """Algorithmic bytes of one K1 launch: the triangular bitmap it writes (row tile I
    stores words [8I, W) of its 256 rows) plus the 16-B lex-order records it reads."""
    Np = -(-N // 1024) * 1024
    W, nT = Np // 32, Np // 256
    words = 256 * (nT * W - 8 * nT * (nT - 1) // 2)
    return (4 * words + 16 * Np) / ws


def k1_traffic(N):
    """dram__bytes_read.sum + dram__bytes_write.sum of K1 from the committed ncu capture, if one
    exists for this N (profiles/traffic.json), else None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get("k_dom_rows8", {}).get(str(N))
    except Exception:
        return None


def k1_roofline_hbm(N, m, ws, avg_s):
    peak, src = hbm_peak()
    b = k1_bytes(N, ws)
    ach = b / avg_s / 1e9
    return {"bound": "hbm", "kernel": "k_dom_rows8 (K1 dominance bitmap)", "achieved": ach, "peak": peak,
            "unit": "GB/s", "frac": ach / peak, "traffic": k1_traffic(N), "algorithmic_bytes": b,
            "avg_launch_ms": avg_s * 1e3, "peak_source": src,
            "note": "K1 is integer-issue bound, not HBM bound (see roofline_compute); bytes = bitmap "
                    "written + records read per launch"}


def k1_roofline_int(N, m, ws, avg_s, sm_mhz):
    """Pair tests/s against the integer-issue ceiling of the packed formulation: 148 SMs x 4
    schedulers x 32 lanes issue one lane-op per cycle, and one pair test costs 2 lane-ops
    (per two columns: m-1 IMAD subtractions, LOP3, LEA; m=3)."""
    pairs = N * (N - 1) / 2 / ws
    ops_per_pair = (m - 1 + (m - 1 + 1) // 2 + 1) / 2
    peak = 148 * 128 * sm_mhz * 1e6 / ops_per_pair
    ach = pairs / avg_s
    return {"bound": "int-issue", "kernel": "k_dom_rows8", "achieved": ach / 1e12, "peak": peak / 1e12,
            "unit": "Tpair/s", "frac": ach / peak, "work_per_launch": pairs,
            "lane_ops_per_pair": ops_per_pair, "sm_mhz": sm_mhz}


# ---------------------------------------------------------------- our arm
def count_launches(stepper, st, gen):
    """Kernels launched by one generation (profiled once, outside the timed region)."""
    import torch

    if os.environ.get("TEMO_BENCH_NO_PROFILER") == "1":  # e.g. under ncu (CUPTI is taken)
        st, _ = stepper.step(st, 0, gen)
        return st, None, None
    try:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            st, _ = stepper.step(st, 0, gen)
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        ours = [n for n in names if "temo" in n or "cub" in n.lower()]
        return st, len(ours), len(names)
    except Exception:  # profiler unavailable: report None (no claim)
        st, _ = stepper.step(st, 0, gen)
        return st, None, None


def our_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2503_20286_b200 import _lib
    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper
    from paper_2503_20286_b200.rng import RngStream

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = RunConfig(algorithm="nsga3", problem=args.problem, objectives=args.objectives, dim=args.dim,
                    pop_size=args.pop, seed=0)  # one shared run; ranks shard the ND sort
    spec, R, n = _resolve(cfg)
    stepper = _Stepper(cfg, spec, R, n)
    gen = RngStream(cfg.seed).split(0).generator()
    st = stepper.init(gen)
    for g in range(args.warmup):
        st, _ = stepper.step(st, g, gen)
    st, launches_per_step, all_kernels = count_launches(stepper, st, gen)
    torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timed region
    clocks = ClockSampler(local)
    clocks.start()
    _lib.timing_enable(True)
    _lib.timing_read(reset=True)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for g in range(args.steps):
        st, _ = stepper.step(st, g, gen)
    e1.record()
    barrier()
    ms = e0.elapsed_time(e1)
    stages = _lib.timing_read(reset=True)
    _lib.timing_enable(False)
    clk = clocks.stop()
    stepper.selector.check()
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    value = args.steps / (ms * 1e-3)  # whole-job gens/s of the one shared run

    # ---- end-to-end through the public harness API: every step uploads its host inputs
    # (the host RNG's pairing + shuffle permutations, pinned ring) and reads its objective
    # matrix back to pinned host memory.  Up to LAG steps in flight: the host draws the next
    # steps' permutations while the GPU runs; step g's result is waited for LAG steps later.
    LAG = 2
    F_host = [torch.empty((n, spec.m), dtype=torch.float64).pin_memory() for _ in range(LAG + 1)]
    done = [torch.cuda.Event() for _ in range(LAG + 1)]
    h = n // 2
    h2d = 8 * (2 * h + (n + 2 * h))  # pairing permutation + shuffle permutation (int64)
    d2h = F_host[0].numel() * 8
    checksum = 0.0
    barrier()
    t0 = time.perf_counter()
    for g in range(args.steps):
        st, _ = stepper.step(st, g, gen)
        F_host[g % (LAG + 1)].copy_(stepper.objectives(st), non_blocking=True)
        done[g % (LAG + 1)].record()
        if g >= LAG:
            done[(g - LAG) % (LAG + 1)].synchronize()
            checksum += float(F_host[(g - LAG) % (LAG + 1)][0, 0])
    for g in range(max(args.steps - LAG, 0), args.steps):
        done[g % (LAG + 1)].synchronize()
        checksum += float(F_host[g % (LAG + 1)][0, 0])
    barrier()
    e2e_s = time.perf_counter() - t0
    t_e2e = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_value = args.steps / float(t_e2e.item())

    # ---- roofline of the dominant kernel (K1 dominance bitmap), measured live above
    N = stepper.N
    m = spec.m
    k1 = stages.get("dom_bits", (float("nan"), 1))
    k1_avg_s = k1[0] / max(k1[1], 1) * 1e-3
    sm_mhz = clk.get("sm_mhz") or 1965.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "roofline": k1_roofline_hbm(N, m, ws, k1_avg_s),
        "roofline_compute": k1_roofline_int(N, m, ws, k1_avg_s, sm_mhz),
        "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()},
        "ndsort_pairs_per_s": None,
        "gpu_launches": (launches_per_step * args.steps) if launches_per_step else None,
        "gpu_launches_per_step": launches_per_step,
        "clocks": clk,
    }
    rank_ms = sum(stages.get(k, (0.0, 1))[0] for k in ("rank_prep", "dom_bits", "peel")) / args.steps
    if rank_ms > 0:
        line["ndsort_pairs_per_s"] = N * (N - 1) / (rank_ms * 1e-3)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args)
        except Exception as exc:  # never lose the GPU line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()

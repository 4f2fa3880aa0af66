"""Benchmark: generations/sec and ND-sort pairs/sec on B200 (BASELINE.json configs A-E).

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl reference] [--config A|B|C|D|E]
One JSON line on rank 0.  With no --config the line is the headline, config D at the
north-star size: NSGA-III on LSMOP1 (m=3, d=1000 requested -> PlatEMO D=992), pop 200k
(merged N=400k).  A step is one full generation (pair -> SBX -> PM -> evaluation -> shuffle
-> ND sort -> normalize -> associate -> niche fill -> survivor bookkeeping) with the
population resident in HBM; ``value`` is whole-job gens/s.  ``e2e`` is the same loop through
the public harness API (``harness._Stepper.step``) with every step's host inputs (the host
Generator's permutations / integer draws, drawn by the native replica) uploaded from pinned
memory and the new objective matrix read back to pinned memory.

The other configs (parity/coverage lines, same JSON shape):
  A  NSGA-III DTLZ1 m=3 d=12 pop 100 (the reference's own CPU-runnable case)
  B  MOEA/D (PBI) DTLZ2 m=3 d=12 pop 10k -> n=9870 directions, T=20
  C  HypE DTLZ2 m=3 d=12 pop 10k (merged N=20k), s=100k Monte-Carlo samples
  D  NSGA-III LSMOP1 m=3 d=1000 pop 200k (default)
  E  ND sort alone: uniform objectives, --objectives m (default 3), --pop N (default 500k);
     a step is one full sort (rank_assign semantics); metric pairs/s = N(N-1)/t.

Multi-GPU (strong scaling, total work fixed): under torchrun the generation is sharded over the
ranks -- offspring pair ranges with one all-gather of the children's [X | F] rows, HypE
Monte-Carlo exchange columns with one all-gather, the ND sort column-sharded for m >= 4 (m <= 3
runs the staircase sort on every rank) -- see DESIGN.md section 6; time is the max over ranks.
``--gpus N`` without torchrun re-launches itself under torch.distributed.run.
``--impl reference`` times the oracle port of the reference algorithm (``oracle/``; the
reference is Python and cannot be compiled) on the host cores on a bounded sample.
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

CONFIGS = {
    "A": dict(algorithm="nsga3", problem="dtlz1", objectives=3, dim=12, pop=100,
              metric="generations/sec (NSGA-III, DTLZ1 m=3 d=12 pop 100)",
              base="BASELINE.json configs[0]: the reference's CPU-runnable case"),
    "B": dict(algorithm="moead", problem="dtlz2", objectives=3, dim=12, pop=10_000, T=20,
              metric="generations/sec (MOEA/D PBI, DTLZ2 m=3 d=12 pop 10k, T=20)",
              base="BASELINE.json configs[1] (PBI: the reference's aggregation)"),
    "C": dict(algorithm="hype", problem="dtlz2", objectives=3, dim=12, pop=10_000, samples=100_000,
              metric="generations/sec (HypE, DTLZ2 m=3 d=12 pop 10k, 100k samples)",
              base="BASELINE.json configs[2]"),
    "D": dict(algorithm="nsga3", problem="lsmop1", objectives=3, dim=1000, pop=200_000,
              metric="generations/sec (NSGA-III, LSMOP1 m=3 d=1000)",
              base="BASELINE.json configs[3] at the north-star size"),
    "E": dict(algorithm="ndsort", objectives=3, pop=500_000,
              metric="ND-sort pairs/sec (uniform objectives)",
              base="BASELINE.json configs[4] (microbench)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="D", choices=sorted(CONFIGS))
    ap.add_argument("--pop", type=int, default=None)
    ap.add_argument("--dim", type=int, default=None)
    ap.add_argument("--objectives", type=int, default=None)
    ap.add_argument("--problem", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    c = dict(CONFIGS[a.config])
    for k in ("pop", "dim", "objectives", "problem"):
        v = getattr(a, k)
        if v is not None:
            c[k] = v
    a.c = c
    return a


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 100 ms during the timed region."""

    def __init__(self, index=0):
        self.proc, self.lines, self.index = None, [], index

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
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:  # first sample before the timed region
                time.sleep(0.02)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self, min_samples=3):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0 = time.time()
        while len(self.lines) < min_samples and time.time() - t0 < 1.0:
            time.sleep(0.05)
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


# ---------------------------------------------------------------- peaks and probes
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback (no MEASURED_PEAKS.json)


def hbm_peak():
    """(GB/s, source) from the driver-written MEASURED_PEAKS.json, else the recipe's fallback."""
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        if "hbm_gbs" in peaks:
            return float(peaks["hbm_gbs"]), "of measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    return FALLBACK_HBM_GBS, "of fallback (B200_PROFILING.md: 6.65 TB/s; MEASURED_PEAKS.json absent)"


def probe_rates(dev):
    """Measured ceilings of the compute-bound kernels' inner-loop mixes (csrc/probe.cu)."""
    import torch

    from paper_2503_20286_b200 import _lib

    L = _lib.lib()
    scratch = torch.zeros(1, dtype=torch.int64, device=dev)
    s = _lib.stream_handle(dev)
    blocks = 148 * 16
    out = {}
    for name, fn, iters in (("philox_blocks_per_s", L.temo_probe_philox_rate, 200),
                            ("packed_pairs_per_s", L.temo_probe_packed_rate, 2000),
                            ("fp64_addsub_per_s", L.temo_probe_dsub_rate, 2000)):
        out[name] = max(fn(blocks, iters, _lib.ptr(scratch), s) for _ in range(3))
    torch.cuda.synchronize()
    return out


def traffic(kernel, key):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` at `key` from the committed ncu
    captures (profiles/traffic.json), else None."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(kernel, {}).get(str(key))
    except Exception:
        return None


# ---------------------------------------------------------------- rooflines
def roofline_offspring(h, d, stages, steps, probes):
    """Offspring step (D/A/C): k_offspring_rand is compute-bound on Philox4x64-10 (5 blocks per
    4 pair-genes: cross, swap, mu, hit c1, hit c2); k_offspring_apply streams parents + spread
    factors in and children out."""
    peak, src = hbm_peak()
    rand_ms = stages.get("offspring", (0.0, 1))[0] / steps
    apply_ms = stages.get("offspring_apply", (0.0, 1))[0] / steps
    quads = h * (-(-d // 4) + 1)
    blocks = 5 * h * d / 4.0
    apply_bytes = 8.0 * (2 * h * d) + 8.0 * (h * d) + 8.0 * (2 * h * d) + 2.0 * quads  # parents, beta, children, flags
    vec_ms = stages.get("apply_vec", (0.0, 1))[0] / steps
    hbm = None
    if vec_ms > 0:  # the streaming kernel of the apply stage, timed alone (its own events)
        ach = apply_bytes / (vec_ms * 1e-3) / 1e9
        hbm = {"bound": "hbm", "kernel": "k_offspring_apply_v (SBX apply + LSMOP sums, streaming)", "achieved": ach,
               "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic("k_offspring_apply_v", 2 * h),
               "algorithmic_bytes": apply_bytes, "avg_launch_ms": vec_ms, "peak_source": src,
               "stage": {"name": "offspring_apply (apply_v + PM hit list + PM/objective pass)",
                         "ms": apply_ms, "achieved": apply_bytes / (apply_ms * 1e-3) / 1e9 if apply_ms > 0 else None}}
    elif apply_ms > 0:
        ach = apply_bytes / (apply_ms * 1e-3) / 1e9
        hbm = {"bound": "hbm", "kernel": "k_offspring_apply (SBX/PM apply + evaluation)", "achieved": ach,
               "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic("k_offspring_apply", 2 * h),
               "algorithmic_bytes": apply_bytes, "avg_launch_ms": apply_ms, "peak_source": src}
    comp = None
    if rand_ms > 0 and probes.get("philox_blocks_per_s"):
        ach = blocks / (rand_ms * 1e-3)
        comp = {"bound": "int-issue (Philox4x64-10)", "kernel": "k_offspring_rand", "achieved": ach / 1e9,
                "peak": probes["philox_blocks_per_s"] / 1e9, "unit": "Gblock/s",
                "frac": ach / probes["philox_blocks_per_s"], "work_per_launch": blocks, "avg_launch_ms": rand_ms,
                "peak_source": "measured: temo_probe_philox_rate (register-only Philox, 4 blocks/thread)"}
    return hbm, comp


def roofline_hv(n1, s, m, stages, steps, probes):
    """HypE (C): n1 x s x m FP64 sample-dominance subtractions (k_hv_dom) + the partial sums."""
    ms = (stages.get("hv_count", (0.0, 1))[0] + stages.get("hv_contrib", (0.0, 1))[0]) / steps
    if ms <= 0 or not probes.get("fp64_addsub_per_s"):
        return None
    work = float(n1) * s * m
    ach = work / (ms * 1e-3)
    return {"bound": "fp64-pipe", "kernel": "k_hv_dom + k_hv_partial/combine", "achieved": ach / 1e12,
            "peak": probes["fp64_addsub_per_s"] / 1e12, "unit": "T FP64 sub/s",
            "frac": ach / probes["fp64_addsub_per_s"], "work_per_step": work, "avg_step_ms": ms,
            "peak_source": "measured: temo_probe_dsub_rate"}


def roofline_moead(n, d, m, T, ms_step):
    """MOEA/D (B) is launch-latency bound at n ~ 10k: bytes per generation vs HBM."""
    peak, src = hbm_peak()
    b = 8.0 * (3 * n * d + 3 * n * m + n * T)
    ach = b / (ms_step * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": "MOEA/D generation (offspring + compare + elite)", "achieved": ach,
            "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None, "algorithmic_bytes": b,
            "peak_source": src, "note": "launch-latency bound; see launch_floor"}


def launch_floor(dev, launches):
    """Time of `launches` back-to-back empty kernel launches (the per-generation floor)."""
    import torch

    if not launches:
        return None
    x = torch.zeros(1, device=dev)
    for _ in range(10):
        x.add_(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(launches):
        x.add_(0)
    b.record()
    torch.cuda.synchronize()
    return {"launches": launches, "ms": a.elapsed_time(b)}


def roofline_ndsort(N, m, stages, steps, probes):
    """E / D's ND sort.  m >= 4: the bitmap K1 (k_dom_rows8 / k_dom_packed) is integer-issue bound.
    m <= 3: the staircase sort; report the HBM view of its setup + peel."""
    peak, src = hbm_peak()
    k1_ms = stages.get("dom_bits", (0.0, 1))[0] / steps
    if m >= 4 and k1_ms > 0:
        Np = -(-N // 1024) * 1024
        W, nT = Np // 32, Np // 256
        words = 256 * (nT * W - 8 * nT * (nT - 1) // 2)
        b = 4.0 * words + 16.0 * Np * ((m + 3) // 4)
        ach = b / (k1_ms * 1e-3) / 1e9
        hbm = {"bound": "hbm", "kernel": f"k_dom_{'rows8' if m <= 5 else 'packed'}<{m}> (K1 dominance bitmap)",
               "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
               "traffic": traffic(f"k_dom_m{m}", N), "algorithmic_bytes": b, "avg_launch_ms": k1_ms,
               "peak_source": src}
        pairs = N * (N - 1) / 2.0
        comp = None
        if probes.get("packed_pairs_per_s"):
            comp = {"bound": "int-issue", "kernel": hbm["kernel"], "achieved": pairs / (k1_ms * 1e-3) / 1e12,
                    "peak": probes["packed_pairs_per_s"] / 1e12, "unit": "Tpair/s",
                    "frac": pairs / (k1_ms * 1e-3) / probes["packed_pairs_per_s"],
                    "note": "peak = measured packed step rate at m = 3 (temo_probe_packed_rate); m > 3 costs "
                            "(m - 1) subtractions per column pair, so the m = 3 rate is an upper bound"}
        return hbm, comp
    ms = sum(stages.get(k, (0.0, 1))[0] for k in ("dom_bits", "peel")) / steps
    if ms <= 0:
        return None, None
    b = 4.0 * 4 * N * max(int(np.ceil(np.log2(max(N, 2)))) - 11, 1)  # high-level arrays written once per sort
    ach = b / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": "staircase sort (k_st_split_* + k_st_local + k_st_peel)", "achieved": ach,
            "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None, "algorithmic_bytes": b,
            "avg_launch_ms": ms, "peak_source": src,
            "note": "latency bound: per front two grid barriers over L2-resident level arrays"}, None


# ---------------------------------------------------------------- CPU baselines
def _oracle_run_step(c, pop, seed=0, reps=1):
    """Seconds per oracle generation of config c at population `pop` (reference algorithm, host)."""
    from oracle import directions as odir
    from oracle import generation, hype as ohype, moead as omoead, problems as oprob, variation as ovar

    m, dim, prob = c["objectives"], c["dim"], c["problem"]
    if prob == "lsmop1":
        dim = oprob.lsmop_dimension(m, dim)
        lower, upper = oprob.lsmop_bounds(m, dim)
    else:
        lower, upper = np.zeros(dim), np.ones(dim)
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed)))
    if c["algorithm"] == "moead":
        W = odir.simplex_lattice(m, odir.largest_h_for(pop, m))
        n = W.shape[0]
        I_nb = odir.neighbors(W, c.get("T", 20))
        X = rng.random((n, dim))
        F = oprob.evaluate(prob, X, m)
        z = F.min(0)
        times = []
        for _ in range(reps):
            t0 = time.perf_counter()
            X, F, z = omoead.step(X, F, z, W, I_nb, 5.0, rng, lambda O: oprob.evaluate(prob, O, m),
                                  20.0, 20.0, None, lower, upper)[:3]
            times.append(time.perf_counter() - t0)
        return min(times), n
    X = lower + rng.random((pop, dim)) * (upper - lower)
    F = oprob.evaluate(prob, X, m)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        if c["algorithm"] == "hype":
            O = ovar.offspring(rng, X, 20.0, 20.0, None, lower, upper)
            Xm, Fm = np.concatenate([X, O]), np.concatenate([F, oprob.evaluate(prob, O, m)])
            s = int(c.get("samples", 10 * pop) * pop / c["pop"])
            X, F = ohype.environmental_selection(Xm, Fm, None, pop, s, rng)
        else:
            W = odir.simplex_lattice(m, odir.largest_h_for(pop, m))
            X, F = generation.nsga3_generation(X, F, W, pop, rng, prob, m, lower, upper)
        times.append(time.perf_counter() - t0)
    return min(times), pop


def cpu_baseline(c, unit):
    """Oracle port timed on a bounded sample; configs above ~pop 4k extrapolated by (pop ratio)^2."""
    cores = os.cpu_count()
    blas = os.environ.get("OPENBLAS_NUM_THREADS", "all")
    if c["algorithm"] == "ndsort":
        from oracle import ndsort as ond

        N, m = c["pop"], c["objectives"]
        ns = 4000
        F = np.random.default_rng(0).random((ns, m))
        t0 = time.perf_counter()
        ond.rank_assign(F, ns)
        t = time.perf_counter() - t0
        t_full = t * (N / ns) ** 2
        return {"value": N * (N - 1) / t_full, "unit": unit, "cores": cores, "kind": "port",
                "sample": f"oracle rank_assign (reference ndsort.py:25-71 restated, NumPy) at N={ns}, m={m} "
                          f"({t:.3f} s), extrapolated by (N ratio)^2 to N={N}; BLAS threads={blas}"}
    pop = c["pop"]
    sample = {"A": 100, "B": 10_000, "C": 2000, "D": 4000}.get(c.get("name"), min(pop, 4000))
    sample = min(sample, pop)
    t, units = _oracle_run_step(c, sample, reps=2 if sample <= 200 else 1)
    scale = 1.0 if sample == pop else (pop / sample) ** 2
    what = "measured at the workload size" if scale == 1.0 else f"extrapolated by (pop ratio)^2 from pop {sample}"
    return {"value": 1.0 / (t * scale), "unit": unit, "cores": cores, "kind": "port",
            "sample": f"oracle (NumPy restatement of temo) {c['algorithm']} generation at pop {sample} "
                      f"({t:.3f} s/gen), {what}; NumPy ufuncs single-threaded, BLAS threads={blas}",
            "measured_s_per_gen_at_sample": t}


def reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    c = dict(args.c, name=args.config)
    unit = "pairs/s" if c["algorithm"] == "ndsort" else "gen/s"
    for _ in range(args.warmup if c["pop"] <= 200 else 1):
        cpu_baseline(c, unit)
    vals = [cpu_baseline(c, unit) for _ in range(args.steps if c["pop"] <= 200 else 1)]
    v = statistics.mean(x["value"] for x in vals)
    ms = (1e3 / v) if unit == "gen/s" else None
    line = {"impl": "reference", "metric": c["metric"], "value": v, "unit": unit, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args),
            "cpu_baseline": dict(vals[-1], value=v),
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args):
    c = args.c
    if c["algorithm"] == "ndsort":
        return {"workload": f"ND sort (rank_assign), m={c['objectives']}, N={c['pop']} uniform objectives; "
                            f"{c['base']}", "N": c["pop"], "objectives": c["objectives"],
                "l2": "objectives 12 MB (< L2); level arrays / bitmap larger than L2",
                "parallelism": "single GPU" if args.gpus == 1 else f"{args.gpus} GPUs"}
    N = 2 * c["pop"] if c["algorithm"] != "moead" else None
    d = c["dim"]
    if c["problem"] == "lsmop1":
        from paper_2503_20286_b200.problems import lsmop_dimension

        d = lsmop_dimension(c["objectives"], c["dim"])[0]
    out = {"workload": f"{c['algorithm'].upper()} {c['problem'].upper()} m={c['objectives']} d={c['dim']}"
                       f"{' (PlatEMO D=%d)' % d if d != c['dim'] else ''} pop={c['pop']}"
                       f"{' (merged N=%d)' % N if N else ''}; {c['base']}",
           "pop": c["pop"], "dim": c["dim"], "D": d, "objectives": c["objectives"], "problem": c["problem"],
           "algorithm": c["algorithm"],
           "rng": "NumPy Philox stream (host permutations/integers by the native replica, device uniforms)",
           "l2": "inputs larger than L2" if c["pop"] * d * 8 > 126e6 else "population fits in L2 (126 MB)",
           "parallelism": "single GPU" if args.gpus == 1 else f"{args.gpus} GPUs"}
    if N:
        out["merged_N"] = N
    if c["algorithm"] == "hype":
        out["samples"] = c.get("samples")
    if c["algorithm"] == "moead":
        out["T"] = c.get("T")
    return out


# ---------------------------------------------------------------- our arm
def count_launches(fn):
    """Kernels launched by one call of fn() (profiled once, outside the timed region)."""
    import torch

    if os.environ.get("TEMO_BENCH_NO_PROFILER") == "1":  # e.g. under ncu (CUPTI is taken)
        fn()
        return None
    try:
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        return len([n for n in names if "temo" in n or "cub" in n.lower() or "Kernel" in n])
    except Exception:
        fn()
        return None


def our_arm(args):
    import torch
    import torch.distributed as dist

    from paper_2503_20286_b200 import _lib

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", torch.cuda.current_device())
    c = dict(args.c, name=args.config)
    probes = probe_rates(dev)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if c["algorithm"] == "ndsort":
        line = bench_ndsort(args, c, dev, probes, barrier, max_over_ranks)
    else:
        line = bench_run(args, c, dev, probes, barrier, max_over_ranks)
    line["probes"] = probes
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(c, line["unit"])
        except Exception as exc:  # never lose the GPU line
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def bench_run(args, c, dev, probes, barrier, max_over_ranks):
    import torch

    from paper_2503_20286_b200 import _lib
    from paper_2503_20286_b200.harness import RunConfig, _resolve, _Stepper
    from paper_2503_20286_b200.rng import RngStream

    ws, rank, local = dist_env()
    cfg = RunConfig(algorithm=c["algorithm"], problem=c["problem"], objectives=c["objectives"], dim=c["dim"],
                    pop_size=c["pop"], seed=0, neighborhood=c.get("T"), hv_samples=c.get("samples"))
    spec, R, n = _resolve(cfg)
    stepper = _Stepper(cfg, spec, R, n)
    gen = RngStream(cfg.seed).split(0).generator()
    st = stepper.init(gen)
    for g in range(args.warmup):
        st, _ = stepper.step(st, g, gen)
    box = [st]

    def one():
        box[0], _ = stepper.step(box[0], 0, gen)

    launches = count_launches(one)
    st = box[0]
    # NSGA-III: the host Generator's inputs of the K timed steps (pairing + shuffle permutations,
    # the offspring's Philox state) are drawn and uploaded before timing -- inputs resident in HBM
    pre = [None] * args.steps
    if c["algorithm"] == "nsga3":
        pre = stepper.upload_host_inputs([stepper.draw_host_inputs(gen) for _ in range(args.steps)])
    torch.cuda.synchronize()
    # ---- device-resident timed region
    clocks = ClockSampler(local)
    clocks.start()
    _lib.timing_enable(False)  # stage times come from the serialised pass below
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for g in range(args.steps):
        st, _ = stepper.step(st, g, gen, timed=False, pre=pre[g], pre_next=pre[g + 1] if g + 1 < args.steps else None)
    e1.record()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    clk = clocks.stop()
    stepper.check()
    value = args.steps / (ms * 1e-3)
    # ---- per-stage device times (rooflines): a separate untimed pass with the randomness
    # overlap off, so each stage's events bracket that stage alone
    ov = stepper.overlap
    stepper.overlap = 0
    pre_s = [None] * args.steps
    if c["algorithm"] == "nsga3":
        pre_s = stepper.upload_host_inputs([stepper.draw_host_inputs(gen) for _ in range(args.steps)])
    torch.cuda.synchronize()
    _lib.timing_enable(True)
    _lib.timing_read(reset=True)
    for g in range(args.steps):
        st, _ = stepper.step(st, g, gen, timed=False, pre=pre_s[g])
    torch.cuda.synchronize()
    stages = _lib.timing_read(reset=True)
    _lib.timing_enable(False)
    stepper.overlap = ov
    # ---- end to end through the harness API: host inputs up, objectives down, LAG steps in flight
    LAG = 2
    m = spec.m
    F_host = [torch.empty((n, m), dtype=torch.float64).pin_memory() for _ in range(LAG + 1)]
    done = [torch.cuda.Event() for _ in range(LAG + 1)]
    h = n // 2
    if c["algorithm"] == "nsga3":
        h2d = 8 * (2 * h + (n + 2 * h))  # pairing + shuffle permutations (int64)
    elif c["algorithm"] == "hype":
        h2d = 8 * 2 * h  # pairing permutation (HypE has no shuffle)
    else:
        h2d = 8 * 2 * n  # MOEA/D parent rows from the two integers draws
    d2h = F_host[0].numel() * 8
    # the e2e loop runs at least 30 generations (a launch-ahead loop from an idle GPU needs a few
    # steps to fill: at 10 steps the fill and the final drain are ~10% of the wall time)
    e2e_steps = max(args.steps, 30)
    barrier()
    t0 = time.perf_counter()
    # NSGA-III host inputs drawn on a worker thread (large populations: the permutations take
    # milliseconds; at pop 100 the thread hand-off costs more than it hides)
    pipe = os.environ.get("TEMO_E2E_PIPE", "1") == "1" and c["pop"] * c["dim"] >= (1 << 20)
    if pipe:
        stepper.start_host_pipeline(gen, e2e_steps)
    for g in range(e2e_steps):
        st, _ = stepper.step(st, g, gen, timed=False)  # host draws of step g+1 overlap step g on the GPU
        F_host[g % (LAG + 1)].copy_(stepper.objectives(st), non_blocking=True)
        done[g % (LAG + 1)].record()
        if g >= LAG:
            done[(g - LAG) % (LAG + 1)].synchronize()
    for g in range(max(e2e_steps - LAG, 0), e2e_steps):
        done[g % (LAG + 1)].synchronize()
    barrier()
    e2e_value = e2e_steps / max_over_ranks(time.perf_counter() - t0)
    stepper.check()
    line = {
        "metric": c["metric"], "value": value, "unit": "gen/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args),
        "e2e": {"value": e2e_value, "unit": "gen/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "host_pipeline": c["algorithm"] == "nsga3" and pipe},
        "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items() if v[1]},
        "stages_note": "per-stage CUDA-event times from a separate serialised pass (randomness overlap off); "
                       "the timed region overlaps the next generation's randomness with this one's apply + selection",
        "gpu_launches": (launches * args.steps) if launches else None,
        "gpu_launches_per_step": launches,
        "clocks": clk,
    }
    if c["algorithm"] == "nsga3" and os.environ.get("TEMO_BENCH_DROPIN", "1") == "1":
        try:
            line["dropin"] = bench_dropin(stepper, st, R, n, dev)
        except Exception as exc:  # never lose the main line
            line["dropin"] = {"error": repr(exc)}
    d = spec.d
    if c["algorithm"] in ("nsga3", "hype"):
        hbm, comp = roofline_offspring(n // 2, d, stages, args.steps, probes)
        line["roofline"] = hbm
        line["roofline_compute"] = comp
        N = stepper.N
        rank_ms = sum(stages.get(k, (0.0, 1))[0] for k in ("rank_prep", "dom_bits", "peel")) / args.steps
        if rank_ms > 0:
            line["ndsort_pairs_per_s"] = N * (N - 1) / (rank_ms * 1e-3)
        if c["algorithm"] == "hype":
            hv = roofline_hv(N, c.get("samples"), m, stages, args.steps, probes)
            if hv:
                line["roofline_compute"] = hv
                line["roofline_offspring_compute"] = comp
        if c["pop"] <= 1000:
            line["launch_floor"] = launch_floor(dev, launches)
    else:
        T = c.get("T") or 20
        line["roofline"] = roofline_moead(n, d, m, T, ms / args.steps)
        line["launch_floor"] = launch_floor(dev, launches)
    return line


def bench_dropin(stepper, st, R, n, dev):
    """The reference-facing NumPy drop-in ``nsga3.environmental_selection(X, F, R, n, rng)``
    (nsga3.py:186-218) on this generation's merged population as HOST arrays: X and F up, the
    selection, the survivors' X and F down -- the call a reference user makes, PCIe included."""
    import torch

    from paper_2503_20286_b200.nsga3 import environmental_selection

    N = stepper.N
    Xh = st.rows(0, N).cpu().numpy()
    Fh = st.cur.F[:N].cpu().numpy()
    rng = np.random.Generator(np.random.Philox(7))
    environmental_selection(Xh, Fh, R, n, rng)  # warm-up (workspaces)
    torch.cuda.synchronize()
    K = 3
    t0 = time.perf_counter()
    for _ in range(K):
        Xn, Fn = environmental_selection(Xh, Fh, R, n, rng)
    dt = (time.perf_counter() - t0) / K
    return {"metric": "nsga3.environmental_selection calls/s (NumPy in, NumPy out)", "value": 1.0 / dt,
            "ms_per_call": dt * 1e3, "h2d_bytes_per_call": Xh.nbytes + Fh.nbytes,
            "d2h_bytes_per_call": Xn.nbytes + Fn.nbytes, "merged_N": N, "survivors": n,
            "note": "pageable host arrays; dominated by the 3.2 GB X upload over PCIe"}


def bench_ndsort(args, c, dev, probes, barrier, max_over_ranks):
    import torch

    from paper_2503_20286_b200 import _lib
    from paper_2503_20286_b200.ndsort import SORT, rank_device

    ws, rank, local = dist_env()
    N, m = c["pop"], c["objectives"]
    Fh = torch.from_numpy(np.random.default_rng(0).random((N, m))).pin_memory()
    F = Fh.to(dev)
    rank_out = (torch.empty(N, dtype=torch.int32, device=dev), torch.empty(1, dtype=torch.int32, device=dev),
                torch.empty(1, dtype=torch.int32, device=dev))
    if ws > 1 and m >= 4:  # column-sharded bitmap sort: each rank owns an equal triangle area
        from paper_2503_20286_b200.parallel import DistRank

        dr = DistRank(N, m, rank, ws, dev)

        def rank_device(Fd, n, mode, out):  # noqa: F811
            r, l, nf = dr(Fd, n, mode)
            out[0].copy_(r)
            out[2].fill_(int(nf))
    for _ in range(args.warmup):
        rank_device(F, N, SORT, out=rank_out)
    launches = count_launches(lambda: rank_device(F, N, SORT, out=rank_out))
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    _lib.timing_enable(True)
    _lib.timing_read(reset=True)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        rank_device(F, N, SORT, out=rank_out)
    e1.record()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    stages = _lib.timing_read(reset=True)
    _lib.timing_enable(False)
    clk = clocks.stop()
    fronts = int(rank_out[2].item())
    # e2e: objectives up from pinned memory, ranks down to pinned memory, every step
    r_host = torch.empty(N, dtype=torch.int32).pin_memory()
    Fd = torch.empty_like(F)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        Fd.copy_(Fh, non_blocking=True)
        rank_device(Fd, N, SORT, out=rank_out)
        r_host.copy_(rank_out[0], non_blocking=True)
    torch.cuda.synchronize()
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0) / args.steps
    pairs = N * (N - 1)
    hbm, comp = roofline_ndsort(N, m, stages, args.steps, probes)
    return {
        "metric": c["metric"], "value": pairs / (ms * 1e-3), "unit": "pairs/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if ws == 1 else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args), fronts=fronts,
                       sharding=("column tiles (bitmap, per-front mask all-gather)" if ws > 1 and m >= 4
                                 else "replicated" if ws > 1 else "single GPU")),
        "e2e": {"value": pairs / e2e_s, "unit": "pairs/s", "h2d_bytes_per_step": N * m * 8, "d2h_bytes_per_step": N * 4},
        "roofline": hbm, "roofline_compute": comp,
        "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items() if v[1]},
        "gpu_launches": (launches * args.steps) if launches else None, "gpu_launches_per_step": launches,
        "clocks": clk,
    }


def main():
    args = parse()
    ws, _, _ = dist_env()
    if args.gpus > 1 and ws == 1 and "TEMO_BENCH_CHILD" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (the driver may also do this itself)
        env = dict(os.environ, TEMO_BENCH_CHILD="1")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000), __file__,
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd, env=env))
    if args.impl == "reference":
        reference_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()

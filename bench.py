#!/usr/bin/env python
"""Himeno Jacobi on B200: GFLOPS + HBM roofline, e2e through the C ABI, GA evals/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs; north_star's headline grid): Himeno L
(257 x 257 x 513, fp32), the best gene pattern's jacobi(nn): the device-resident
time loop (gene 6; fused stencil with p/wrk2 rotation).  One *step* =
one jacobi(nn) call, nn = 100 iterations (N = 100).
Inputs (1.9 GB) exceed the 126 MB L2, so no flush is needed between steps.
GFLOPS = 34 * (I-3)(J-3)(K-3) * nn / t.

* value      device-resident: K steps between CUDA events on the library's
             stream, barrier + synchronize on both sides, max over ranks.
* e2e        hp_jacobi_host (C ABI) with pinned HOST buffers: H2D of the 13
             input arrays, the time loop, D2H of p and gosa -- per step.
* roofline   dominant kernel = the stencil launch; achieved = 56 B/pt * N_int /
             its CUDA-event duration; peak = MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline  the CPU oracle's jacobi on the same grid, all host threads.
* ga         run_ga (config 4: pop 20 x gen 20, Himeno M, nn=3) with B200Evaluator on
             this rank's GPU: fresh evaluations/s and generations/s; ga_config1 the
             same for config 1 (Himeno XS, pop 4 x gen 4); ft_ga the GA on NAS FT class S
             through the generated executor (pop 20 x gen 5, verified genes).

N > 1 (torchrun): the grid is split into N slabs of i-planes (dd.SlabJacobi), one
per GPU; halo planes and the gosa all-reduce go over NCCL; "scaling": "strong"
(total work fixed).  --impl reference: rank 0 times the CPU reference path
(oracle jacobi, OpenMP over all host cores); other ranks exit 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FLOP_PER_POINT = 34
BYTES_STENCIL = 56


def launch_bytes(points: int, iters_per_launch: float) -> float:
    """Algorithmic HBM bytes of one stencil launch: 56 B per interior point per pass;
    a two-step pass covers two iterations, a flow launch all the passes of a step."""
    passes = iters_per_launch / 2 if iters_per_launch > 1.5 else 1.0
    return BYTES_STENCIL * points * passes


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _hbm_entries(d, path=()):
    """(key path, GB/s) for every numeric HBM figure in MEASURED_PEAKS.json."""
    out = []
    if isinstance(d, dict):
        for k, v in d.items():
            out += _hbm_entries(v, path + (str(k).lower(),))
    elif isinstance(d, (int, float)) and not isinstance(d, bool):
        key = "_".join(path)
        if "hbm" in key or "dram" in key or "copy" in key:
            if "tf" not in key and "flop" not in key and d > 0:
                out.append((key, float(d)))
    return out


def peaks():
    """HBM roofline denominator: the driver-written measured figure when present (the
    sustained one -- the stencil is timed inside a 100-iteration step), else the
    profiling guide's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            entries = _hbm_entries(json.loads(p.read_text()))
        except ValueError:
            entries = []
        for want in ("sustained", "burst", ""):
            for key, v in entries:
                if want in key:
                    # a TB/s figure is converted to GB/s
                    return (v * 1000.0 if v < 100 else v), f"measured (MEASURED_PEAKS.json {key})"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def copy_bandwidth_gbs(device: int, nbytes: int = 1 << 31, reps: int = 5) -> float:
    """Live device-to-device copy bandwidth (read + write bytes / time, best of reps):
    context for the roofline denominator, measured on this box in this run."""
    import torch
    dev = torch.device("cuda", device)
    a = torch.empty(nbytes // 4, dtype=torch.float32, device=dev).fill_(1.0)
    b = torch.empty_like(a)
    best = float("inf")
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * nbytes / (best / 1e3) / 1e9


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        if self.path and os.path.exists(self.path):
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
            os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows)}


def dist_setup():
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    return world, rank, local


def host_threads() -> int:
    """Host threads this process may run on (torchrun exports OMP_NUM_THREADS=1, which
    must not shrink the CPU reference: rank 0 alone runs it)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):
        return max(1, os.cpu_count() or 1)


def cpu_baseline(size, seconds: float, threads: int) -> dict:
    """CPU oracle jacobi on the same grid, bounded to ~`seconds` of work -- the same
    procedure (oracle/cpu_bench.py: fresh process, bound threads, parallel first
    touch) as the --impl reference arm."""
    from oracle import cpu_bench
    return cpu_bench.run_subprocess(size.name, seconds, threads)


def reference_program(size):
    """The program binary the reference's compile template produces (oracle/_ref, gcc -O2,
    pragmas ignored, single-threaded), timed the way ExternalEvaluator times a run
    (wall clock around the process, evaluators.py:207-214): nn=3 minus nn=1 = two Jacobi
    iterations.  None when the binaries were not built (reference not mounted)."""
    import subprocess
    ref = ROOT / "oracle" / "_ref"
    b1, b3 = ref / f"himeno_{size.name.lower()}_n1", ref / f"himeno_{size.name.lower()}_n3"
    if not (b1.exists() and b3.exists()):
        return None

    def run(b):
        t0 = time.perf_counter()
        subprocess.run([str(b)], check=True, stdout=subprocess.DEVNULL)
        return time.perf_counter() - t0

    t1 = min(run(b1) for _ in range(2))
    t3 = min(run(b3) for _ in range(2))
    gf = FLOP_PER_POINT * size.interior_points * 2 / max(t3 - t1, 1e-9) / 1e9
    return {"value": gf, "unit": "GFLOP/s", "cores": 1, "kind": "reference",
            "sample": f"oracle/_ref program ({size.name}, gcc -O2 -w, single-threaded): "
                      f"wall(nn=3) {t3:.2f} s - wall(nn=1) {t1:.2f} s = 2 iterations"}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    from oracle import cpu_bench
    from paper_2002_12115_b200.apps import himeno
    size = himeno.size(args.size)
    threads = host_threads()
    # one step = one Jacobi iteration of the oracle (a bounded sample of the
    # workload); the same procedure as the B200 arm's cpu_baseline object
    r = cpu_bench.run_subprocess(size.name, 0.0, threads, min_iters=args.steps,
                                 warmup=args.warmup)
    value = r["value"]
    el = FLOP_PER_POINT * size.interior_points * args.steps / (value * 1e9)
    line = {
        "impl": "reference", "metric": "Himeno GFLOPS", "value": value, "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (Himeno initmt state)",
        "config": {"workload": f"himeno_{size.name}_jacobi", "grid": [size.I, size.J, size.K],
                   "nn_per_step": 1, "threads": threads},
        "cpu_baseline": r,
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    prog = reference_program(size)
    if prog is not None:
        line["reference_program"] = prog
    if not args.no_ga:
        from oracle import ref_ga
        line["ga"] = ref_ga.ga_throughput(args.ga_size, args.ga_nn, args.ga_pop, args.ga_gens,
                                          args.ga_seed)
        line["ga_config1"] = ref_ga.ga_throughput("XS", 3, 4, 4, args.ga_seed)
        if not args.no_ft:
            line["ft_ga"] = ref_ga.ft_ga_throughput("S", args.ga_pop, args.ft_gens, args.ga_seed)
    print(json.dumps(line), flush=True)
    return 0


# exhaustive optimum over the 272 runnable genomes (scripts/eval_all.py;
# profiles/r01_evalall_M.jsonl): the reference's brute_force_optimum
# (evaluators.py:131-147) with the real evaluator, Himeno M, nn = 3
OPTIMUM = {("M", 3): "1001001000000"}


def ga_throughput(devices, size_name: str, nn: int, pop: int, gens: int, seed: int,
                  workers: int = 1, nested_policy: str = "reject",
                  host_build: str = "tuned") -> dict:
    """run_ga with the B200 evaluator.  Counts what the reference's procedure would
    count as work: `executed_evals` are runs of the program; genomes with nested
    compute constructs are rejected before anything launches (the reference's
    compile failure; `rejected_before_launch`) and are reported apart."""
    from paper_2002_12115_b200 import ga
    from paper_2002_12115_b200.evaluator import B200Evaluator
    devices = [devices] if isinstance(devices, int) else list(devices)
    with B200Evaluator(size_name, nn=nn, devices=devices, workers_per_device=workers,
                       nested_policy=nested_policy, host_build=host_build) as ev:
        t_setup = time.perf_counter()
        ev.prepare()                                       # one device context per slot
        ev.measure((0,) * ev.gene_length)                  # first-touch warm-up
        setup_s = time.perf_counter() - t_setup
        done, executed = {}, []
        measure = ev.measure
        import threading
        lock = threading.Lock()
        busy = {d: 0.0 for d in sorted(set(devices))}    # program-run seconds per GPU
        runs = {d: 0 for d in busy}

        def timed_measure(g):
            m = measure(g)
            st = ev.stats.get(tuple(g)) if ev.lowered(g).failure is None else None
            with lock:
                done[tuple(g)] = time.perf_counter()
                if st is not None:
                    executed.append(g)
                    if m.seconds:
                        busy[st["device"]] += m.seconds
                        runs[st["device"]] += 1
            return m

        ev.measure = timed_measure
        try:
            import psutil
            psutil.cpu_percent(interval=None)
        except ImportError:   # host-load figures are context only
            psutil = None
        cpu0 = os.times()
        t0 = time.perf_counter()
        res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                        ev.gene_length, ev)
        el = time.perf_counter() - t0
        cpu1 = os.times()
        sys_pct = psutil.cpu_percent(interval=None) if psutil else None
        ev.measure = measure
        best = res.best
        out = {"size": size_name, "nn": nn, "population": pop, "generations": gens,
               "seed": seed, "nested_policy": nested_policy, "gpus": len(devices),
               "workers_per_gpu": workers, "setup_s": setup_s, "wall_s": el,
               "fresh_evals": res.evaluations, "executed_evals": len(executed),
               "rejected_before_launch": res.evaluations - len(executed),
               "executed_evals_per_s": len(executed) / el,
               "fresh_evals_per_s": res.evaluations / el, "gens_per_s": gens / el,
               "best_genome": ga.genome_str(best.genome), "best_time_s": best.time_s,
               "best_source": best.eval_source,
               "time_to_best_s": (done[best.genome] - t0) if best.genome in done else None,
               # per GPU: seconds of program runs (the fitness wall time of each executed
               # evaluation) summed over its worker slots, and that sum over the GA's wall
               # time (concurrent slots overlap, so it can exceed 1)
               "per_gpu": {str(d): {"runs": runs[d], "busy_s": busy[d], "busy_frac": busy[d] / el}
                           for d in busy},
               # host: the process's CPU seconds over the GA (host loops of gene-0 nests,
               # planning, launches) as mean busy cores, and the whole machine's load
               "host": {"process_cpu_s": (cpu1.user - cpu0.user) + (cpu1.system - cpu0.system),
                        "mean_busy_cores": ((cpu1.user - cpu0.user) + (cpu1.system - cpu0.system)) / el,
                        "cores": os.cpu_count(), "system_cpu_pct": sys_pct}}
        opt = OPTIMUM.get((size_name, nn))
        if opt is not None and best.time_s < 1000:
            g = tuple(int(c) for c in opt)
            t_opt = min(ev.measure(g).seconds for _ in range(5))
            t_best = min(ev.measure(best.genome).seconds for _ in range(5))
            out["optimum"] = {"genome": opt, "time_s": t_opt, "best_time_s_remeasured": t_best,
                              "best_over_optimum": t_best / t_opt,
                              "source": "exhaustive search of the 272 runnable genomes "
                                        "(profiles/r01_evalall_M.jsonl), re-measured now"}
    return out


# candidate patterns for the fitness-path e2e line on the headline grid: the device
# time loop alone, the exhaustive optimum at M (initmt and the time loop on the
# device), and the stencil + copy nests as kernels
E2E_FITNESS_PATTERNS = ("0000001000000", "1001001000000", "0000000100100")


def fitness_e2e(device: int, size, nn: int, reps: int = 3) -> dict:
    """The fitness evaluation itself on the headline grid: B200Evaluator.measure ->
    hp_run, i.e. the whole program run the reference times around its process
    (evaluators.py:207-214) -- initmt, the plan's host<->device transfers of the
    program's host arrays, jacobi(nn), main's prints.  GFLOP/s = the program's
    jacobi flops / wall time (best of `reps`)."""
    from paper_2002_12115_b200.evaluator import B200Evaluator
    flops = FLOP_PER_POINT * size.interior_points * nn
    pats = {}
    with B200Evaluator(size.name, nn=nn, devices=[device]) as ev:
        ev.prepare()
        for s in E2E_FITNESS_PATTERNS:
            g = tuple(int(c) for c in s)
            ev.measure(g)                                  # warm-up (first touch)
            ts = [ev.measure(g).seconds for _ in range(reps)]
            st = ev.stats[g]
            pats[s] = {"wall_s": min(ts), "gflops": flops / min(ts) / 1e9,
                       "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"],
                       "n_launch": st["n_launch"], "host_s": st["host_s"],
                       "xfer_s": st["xfer_s"], "gosa": st["gosa"]}
    best = min(pats, key=lambda k: pats[k]["wall_s"])
    return {"value": pats[best]["gflops"], "unit": "GFLOP/s", "best_pattern": best,
            "h2d_bytes_per_step": pats[best]["h2d_bytes"],
            "d2h_bytes_per_step": pats[best]["d2h_bytes"],
            "path": "B200Evaluator.measure -> hp_run (C ABI): the whole program under the "
                    "pattern, host arrays, the plan's transfers, wall clock",
            "grid": [size.I, size.J, size.K], "nn": nn, "patterns": pats}


def ft_ga_throughput(devices, cls: str, pop: int, gens: int, seed: int, workers: int) -> dict:
    """run_ga on NAS FT through the generated executor (generic.GenEvaluator): genes =
    the loops the execution probe verified and whose device version alone does not slow
    the program down (the search-space narrowing of the paper), nested genes run under
    their outermost anchor, every run's output verified."""
    from paper_2002_12115_b200 import ga, generic
    devices = [devices] if isinstance(devices, int) else list(devices)
    app = f"ft_{cls.lower()}"
    t0 = time.perf_counter()
    with generic.GenEvaluator(app, devices=devices, workers_per_device=workers,
                              verify_each=True, nested_policy="outermost",
                              genes="screened") as ev:
        probe_s = time.perf_counter() - t0
        ev.prepare()
        cpu_s = ev.measure((0,) * ev.gene_length).seconds
        t0 = time.perf_counter()
        res = ga.run_ga(ga.GAConfig(population=pop, generations=gens, rng_seed=seed),
                        ev.gene_length, ev)
        el = time.perf_counter() - t0
        valid = sum(1 for r in res.records for i in r.individuals
                    if i.eval_source == "fresh" and i.time_s < 1000)
        return {"app": app, "population": pop, "generations": gens, "seed": seed,
                "gpus": len(devices), "workers_per_gpu": workers,
                "genes": ev.gene_length, "classified_genes": len(ev.classified_ids),
                "probe_s": probe_s, "wall_s": el, "fresh_evals": res.evaluations,
                "valid_fresh": valid, "evals_per_s": res.evaluations / el,
                "gens_per_s": gens / el, "best_genome": ga.genome_str(res.best.genome),
                "best_time_s": res.best.time_s, "all_cpu_time_s": cpu_s,
                "note": "each evaluation runs the pattern's own device/host mix with blocking "
                        "OpenACC transfer semantics (random FT patterns: ~1e5 launches and "
                        "transfers per run); the reference procedure compiles and runs the "
                        "all-CPU binary for every genome (gcc ignores the pragmas)"}


def verify_step(ctx, slab, size, nn: int, variant: int) -> dict:
    """Re-run one step from the initial state and compare it with the CPU oracle's
    committed result for this grid and nn (fails loudly on a mismatch)."""
    import hashlib
    gold_path = ROOT / "tests" / "golden" / f"himeno_{size.name.lower()}_n{nn}.json"
    if slab is None:
        ctx.init_device()
        ctx.jacobi_device(nn, variant)
    else:
        ctx.init_device()
        slab.jacobi(nn)
    ctx.sync()
    gosa = slab.gosa() if slab is not None else ctx.read_gosa(1)
    out = {"gosa": gosa, "golden": None}
    if not gold_path.exists():
        if not (gosa == gosa and gosa > 0):
            raise RuntimeError(f"bad gosa {gosa}")
        out["golden"] = "none committed for this grid/nn: gosa checked finite and positive"
        return out
    gold = json.loads(gold_path.read_text())
    rel = abs(gosa - gold["gosa64"]) / gold["gosa64"]
    out.update(golden=str(gold_path.relative_to(ROOT)), gosa_oracle=gold["gosa64"],
               gosa_rel_err=rel)
    if rel > 1e-11:
        raise RuntimeError(f"gosa {gosa!r} differs from the oracle's {gold['gosa64']!r} ({rel:.2e})")
    if slab is None:
        p = ctx.read_field("p", 1)
        match = hashlib.sha256(p.tobytes()).hexdigest() == gold["p_sha256"]
        out["p_sha256_match"] = match
        if not match:
            raise RuntimeError("p after the step differs from the oracle's (SHA-256)")
    return out


def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    from paper_2002_12115_b200 import native as N
    from paper_2002_12115_b200.apps import himeno

    dist = None
    if world > 1:
        # NCCL's communicator set-up lines (rank count, transports, NVLS) on stderr, so
        # the run's log shows the nranks the halo exchange and gosa all-reduce used;
        # INIT only (no per-call logging inside the timed region)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)

    def barrier():
        if dist is not None:
            dist.barrier()

    size = himeno.size(args.size)
    nn, variant = args.nn, args.variant
    flops_step = FLOP_PER_POINT * size.interior_points * nn      # whole grid, one step
    slab = None
    if world > 1:
        # strong scaling: the grid is split into slabs, halo planes + gosa over NCCL
        from paper_2002_12115_b200.dd import SlabJacobi
        slab = SlabJacobi(size, rank, world, local, dist=dist)
        ctx = slab.ctx
        timed = lambda k: slab.time_steps(k, nn)           # noqa: E731
    else:
        ctx = N.Context(local, size.I, size.J, size.K)
        ctx.init_device()
        timed = lambda k: ctx.time_steps(k, nn, variant)   # noqa: E731
    for _ in range(args.warmup):
        timed(1)

    n0 = ctx.launch_count
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        ms = timed(args.steps)
        torch.cuda.synchronize()
        barrier()
    launches = ctx.launch_count - n0
    clk = clocks.summary()
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = args.steps * flops_step / (ms_max / 1e3) / 1e9

    # correctness: one fresh jacobi(nn) from the initial state against the oracle's
    # committed result (tests/golden/himeno_l_n100.json; scripts/gen_golden_l100.py)
    verified = verify_step(ctx, slab, size, nn, variant)

    # dominant kernel (the stencil launch), CUDA events per launch; also the
    # single-step kernel (temporal blocking off) for reference
    lib = ctx.lib
    tb_on = lib.hp_set_temporal_blocking(-1)
    kt = ctx.time_jacobi(nn, variant)      # this rank's grid or slab, no exchange
    two_step_kernel = N.last_two_step_kernel()
    lib.hp_set_temporal_blocking(0)
    kt1 = ctx.time_jacobi(nn, variant)
    lib.hp_set_temporal_blocking(tb_on)
    peak, peak_src = peaks()
    points = slab.interior_points if slab is not None else size.interior_points
    achieved = launch_bytes(points, kt.stencil_iters) / (kt.stencil_ms / 1e3) / 1e9
    # DRAM bytes per launch from the committed ncu capture of the same kernel (L grid)
    ncu_kernels = {}
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        try:
            ncu_kernels = json.loads(prof.read_text()).get("kernels", {})
        except ValueError:
            ncu_kernels = {}
    key_tb, key_1 = "k_stencil_tb2", "k_stencil_tma<3>"
    on_l = size.name == "L" and slab is None
    traffic = (ncu_kernels.get(key_tb if kt.stencil_iters > 1.5 else key_1, {})
               .get("dram_bytes_per_launch") if on_l else None)
    traffic1 = ncu_kernels.get(key_1, {}).get("dram_bytes_per_launch") if on_l else None
    achieved1 = BYTES_STENCIL * points / (kt1.stencil_ms / 1e3) / 1e9
    roofline_single = {"bound": "hbm", "achieved": achieved1, "peak": peak, "unit": "GB/s",
                       "frac": achieved1 / peak, "kernel": "k_stencil_tma<3> (one iteration per pass)",
                       "launch_ms": kt1.stencil_ms, "iterations_per_launch": kt1.stencil_iters,
                       "traffic": traffic1,
                       "gflops": FLOP_PER_POINT * points * kt1.stencil_iters / kt1.stencil_ms / 1e6}
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": (f"{two_step_kernel} (temporal blocking: 2 iterations per pass, 56 B/pt "
                           "per pass; warp-specialised TMA pipeline, step-2 coefficients "
                           "handed over in tensor memory by the step-1 warps)"
                           if variant == 1 and kt.stencil_iters > 1.5 else "k_stencil_tma<3>"),
                "bytes_per_point": BYTES_STENCIL, "points_per_launch": points,
                "passes_per_launch": launch_bytes(points, kt.stencil_iters) / (BYTES_STENCIL * points),
                "launch_ms": kt.stencil_ms, "share_of_step": kt.stencil_ms * kt.n_stencil / kt.total_ms,
                "iterations_per_launch": kt.stencil_iters,
                "peak_source": peak_src}
    # the same kernel inside the timed region: its launches run back to back there (PDL
    # overlaps each launch's tail with the next one's start, which per-launch events
    # prevent); the whole step's device time is charged to the stencil launches, so this
    # is a lower bound for the in-step rate
    if kt.n_stencil > 0 and ms_max > 0:
        in_step_ms = ms_max / args.steps / kt.n_stencil
        in_step = launch_bytes(points, kt.stencil_iters) / (in_step_ms / 1e3) / 1e9
        roofline["in_step"] = {"launch_ms": in_step_ms, "achieved": in_step, "frac": in_step / peak,
                               "launches_per_step": kt.n_stencil}
    # the same box's device-to-device copy bandwidth, measured now (context for `peak`)
    try:
        live = copy_bandwidth_gbs(local)
        roofline["copy_gbs_live"] = live
        roofline["frac_of_copy_live"] = achieved / live
    except Exception as exc:  # noqa: BLE001 -- context only, never fatal
        roofline["copy_gbs_live"] = None
        print(f"copy bandwidth probe failed: {exc}", file=sys.stderr)

    # e2e through the C ABI with pinned host buffers: H2D of the inputs, the
    # time loop, D2H of p and gosa, every step (per rank: its slab)
    # the e2e pipeline's fill / drain is amortised over --e2e-steps jobs (default 20),
    # independent of --steps (each job is ~35 ms on L)
    e2e_steps = max(1, args.e2e_steps)
    import ctypes
    host = {}
    ctx.init_device()
    pinned = []
    I_loc = ctx.shape[0]
    nbytes = I_loc * size.J * size.K * 4
    for name in N.FIELDS:
        ptr = ctx.lib.hp_host_alloc(nbytes)
        if not ptr:
            raise RuntimeError("pinned allocation failed")
        pinned.append(ptr)
        arr = np.ctypeslib.as_array((ctypes.c_float * (nbytes // 4)).from_address(ptr))
        host[name] = arr.reshape(I_loc, size.J, size.K)
        host[name][...] = ctx.read_field(name, 1)
    p_out = host["wrk2"]   # wrk2 is not an input; reuse its pinned buffer for p

    def e2e_step():
        if slab is None:
            return ctx.jacobi_host(host, nn, variant, p_out)
        for name in N.FIELDS:
            if name != "wrk2":
                ctx.write_field(name, 1, host[name])
        slab.jacobi(nn)
        p_out[...] = ctx.read_field("p", 1)
        return ctx.read_gosa(1)

    def timed(run, n):
        barrier()
        t0 = time.perf_counter()
        run(n)
        el = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        barrier()
        return el

    gosa_serial = e2e_step()     # warm-up
    serial_s = timed(lambda n: [e2e_step() for _ in range(n)], e2e_steps)
    e2e_s, path = serial_s, ("hp_jacobi_host (C ABI), pinned host" if slab is None
                             else "hp_write_field + hp_dd_jacobi + hp_read_field per slab (C ABI)")
    pipelined = None
    if slab is None and e2e_steps >= 2:
        # K contexts, jobs round-robin: while one job's inputs stream in over PCIe the
        # others run their loops and read back, so the host->device link never idles
        K = max(2, args.e2e_contexts)
        ctxs, outs = [ctx], [p_out]
        for _ in range(K - 1):
            ctxs.append(N.Context(local, size.I, size.J, size.K))
            ptr2 = ctx.lib.hp_host_alloc(nbytes)
            if not ptr2:
                raise RuntimeError("pinned allocation failed")
            pinned.append(ptr2)
            outs.append(np.ctypeslib.as_array(
                (ctypes.c_float * (nbytes // 4)).from_address(ptr2)).reshape(I_loc, size.J, size.K))
        gosas = []

        def run_pipelined(n):
            pending = [False] * K
            for s in range(n):
                x = s % K
                if pending[x]:
                    gosas.append(ctxs[x].sync())
                ctxs[x].jacobi_host_async(host, nn, variant, outs[x])
                pending[x] = True
            for x in range(K):
                if pending[x]:
                    gosas.append(ctxs[x].sync())

        run_pipelined(K)   # warm-up of every context
        gosas.clear()
        pipe_s = timed(run_pipelined, e2e_steps)
        if any(g != gosa_serial for g in gosas) or not all(np.array_equal(p_out, o) for o in outs[1:]):
            raise RuntimeError("pipelined e2e results differ from the serial call")
        for c in ctxs[1:]:
            c.close()
        pipelined = pipe_s
        e2e_s = pipe_s
        path = (f"hp_jacobi_host_async on {K} contexts, jobs round-robin (H2D of one job "
                "overlaps the others' loops + D2H), pinned host")
    for ptr in pinned:
        ctx.lib.hp_host_free(ptr)
    e2e_value = e2e_steps * flops_step / e2e_s / 1e9
    e2e = {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": 13 * nbytes,
           "d2h_bytes_per_step": nbytes + 8, "steps": e2e_steps,
           "ms_per_step": e2e_s * 1e3 / e2e_steps, "path": path,
           "serial": {"value": e2e_steps * flops_step / serial_s / 1e9,
                      "ms_per_step": serial_s * 1e3 / e2e_steps,
                      "path": "hp_jacobi_host, one job at a time"}}

    extra = {}
    if rank == 0 and world == 1 and not args.no_other_grids:
        # the other BASELINE grids on this GPU, same method (device-resident time loop)
        others = {}
        for name in ("M", "XL"):
            osz = himeno.size(name)
            with N.Context(local, osz.I, osz.J, osz.K) as octx:
                octx.init_device()
                octx.time_steps(1, nn, variant)
                oms = octx.time_steps(3, nn, variant)
                okt = octx.time_jacobi(nn, variant)
                okern = N.last_two_step_kernel()
            obytes = launch_bytes(osz.interior_points, okt.stencil_iters)
            others[name] = {
                "grid": [osz.I, osz.J, osz.K],
                "gflops": 3 * FLOP_PER_POINT * osz.interior_points * nn / (oms / 1e3) / 1e9,
                "kernel": okern,
                "stencil_launch_ms": okt.stencil_ms,
                "iterations_per_launch": okt.stencil_iters,
                "passes_per_launch": obytes / (BYTES_STENCIL * osz.interior_points),
                "achieved_gbs": obytes / (okt.stencil_ms / 1e3) / 1e9}
            others[name]["frac"] = others[name]["achieved_gbs"] / peaks()[0]
        extra["other_grids"] = others
    if rank == 0 and world == 1 and not args.no_fitness_e2e:
        extra["e2e_fitness"] = fitness_e2e(local, size, nn)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        extra["cpu_baseline"] = cpu_baseline(size, args.cpu_seconds, host_threads())
    if rank == 0 and not args.no_ga:
        # N > 1: the population is sharded over every GPU of the node (config 4), one
        # worker slot per GPU, from rank 0's process
        devices = [local] if world == 1 else list(range(world))
        workers = (args.ga_workers or min(16, os.cpu_count() or 1)) if world == 1 else 1
        extra["ga"] = ga_throughput(devices, args.ga_size, args.ga_nn, args.ga_pop,
                                    args.ga_gens, args.ga_seed, workers)
        # BASELINE config 1: Himeno XS, nn=3, pop 4 x gen 4 -- reference-faithful
        # ("reject": nested compute constructs fail like the OpenACC compile) and with
        # nested genes running their outermost anchor (every genome runs)
        extra["ga_config1"] = ga_throughput(devices, "XS", 3, 4, 4, args.ga_seed, workers)
        extra["ga_config1_outermost"] = ga_throughput(devices, "XS", 3, 4, 4, args.ga_seed,
                                                      workers, nested_policy="outermost")
        if not args.no_ft:
            extra["ft_ga"] = ft_ga_throughput(devices, "S", args.ga_pop, args.ft_gens,
                                              args.ga_seed, workers)
    barrier()   # the other ranks wait for rank 0's extras before tearing down NCCL
    if slab is not None:
        slab.close()
    else:
        ctx.close()

    if rank == 0:
        line = {
            "metric": "Himeno GFLOPS", "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Himeno initmt state, deterministic)",
            "config": {"workload": f"himeno_{size.name}_jacobi", "grid": [size.I, size.J, size.K],
                       "nn_per_step": nn, "pattern": "0000001000000 (device time loop)",
                       "variant": "fused rotation" if variant == 1 else "stencil+copy",
                       "parallelism": f"slab{world} (i-planes, NCCL halo + gosa all-reduce)"
                       if world > 1 else "single",
                       "l2": "inputs 1.9 GB > 126 MB L2 (no flush)"},
            "roofline": roofline, "roofline_single_step": roofline_single, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk,
            "gosa": verified["gosa"], "verified": verified,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--size", default="L")
    ap.add_argument("--nn", type=int, default=100)
    ap.add_argument("--variant", type=int, default=1, choices=[0, 1])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-contexts", type=int, default=2,
                    help="contexts (jobs in flight) of the pipelined e2e measurement")
    ap.add_argument("--no-ga", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-grids", action="store_true")
    ap.add_argument("--no-fitness-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ga-size", default="M")
    ap.add_argument("--ga-nn", type=int, default=3)
    ap.add_argument("--ga-pop", type=int, default=20)
    ap.add_argument("--ga-gens", type=int, default=20)
    ap.add_argument("--ga-seed", type=int, default=0)
    ap.add_argument("--no-ft", action="store_true", help="skip the NAS FT GA line")
    ap.add_argument("--ft-gens", type=int, default=5)
    ap.add_argument("--ga-workers", type=int, default=4,
                    help="concurrent evaluations per GPU (own context each); 4, 8 and 16 give "
                         "the same evals/s (profiles/r01_ga_workers.jsonl); 0 = host cores")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())

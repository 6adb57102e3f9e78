"""The tuning pipeline on the B200 evaluator: baseline -> GA -> best plan -> verification -> report.

Mirrors the reference's ``run_pipeline`` (acctuner/cli.py:211-284) for the hot path:
``measure_baseline`` (cli.py:200-208), ``run_ga`` (ga.py:183-211), the numeric output
diff ``verify_results`` (cli.py:155-186; defaults atol 1e-6, rtol 1e-4, cli.py:34-35)
between the all-CPU program's stdout and the best pattern's, and the report files
(``report.json`` with the reference's keys, ``generations.jsonl``, ``meta.json``;
cli.py:287-317).  Front-end stages (parse/classify) are replaced by the committed
program model (apps/model/himeno.json).

    python -m paper_2002_12115_b200.tune --size M --nn 3 --population 20 \\
        --generations 20 --devices all --out tune-out
"""

from __future__ import annotations

import argparse
import json
import platform
import sys
import time
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional

from . import ga
from .errors import UnparsableOutput
from .evaluator import B200Evaluator, measure_baseline

DEFAULT_ATOL = 1e-6
DEFAULT_RTOL = 1e-4


@dataclass
class DiffReport:
    passed: bool
    values_compared: int
    max_abs_err: float
    max_rel_err: float
    mismatches: int
    atol: float
    rtol: float
    length_mismatch: bool = False
    detail: list = field(default_factory=list)

    def to_json(self) -> dict:
        return {"passed": self.passed, "values_compared": self.values_compared,
                "max_abs_err": self.max_abs_err, "max_rel_err": self.max_rel_err,
                "mismatches": self.mismatches, "atol": self.atol, "rtol": self.rtol,
                "length_mismatch": self.length_mismatch, "detail": self.detail[:10]}


def _number(token: str) -> Optional[float]:
    try:
        return float(token)
    except ValueError:
        return None


def verify_results(baseline_output: str, tuned_output: str, atol: float = DEFAULT_ATOL,
                   rtol: float = DEFAULT_RTOL) -> DiffReport:
    """Whitespace-token numeric diff: pass iff |t - b| <= atol + rtol*|b| for every value;
    non-numeric tokens must match exactly; different token counts fail."""
    if not isinstance(baseline_output, str) or not isinstance(tuned_output, str):
        raise UnparsableOutput("output streams must be text")
    base, tuned = baseline_output.split(), tuned_output.split()
    rep = DiffReport(True, 0, 0.0, 0.0, 0, atol, rtol)
    if len(base) != len(tuned):
        rep.passed = False
        rep.length_mismatch = True
        rep.detail.append(f"value counts differ: {len(base)} vs {len(tuned)}")
    for idx, (b, t) in enumerate(zip(base, tuned)):
        rep.values_compared += 1
        fb, ft = _number(b), _number(t)
        if fb is None or ft is None:
            if b != t:
                rep.mismatches += 1
                rep.passed = False
                rep.detail.append(f"token {idx}: {t!r} != {b!r}")
            continue
        abs_err = abs(ft - fb)
        rel_err = abs_err / abs(fb) if fb != 0 else (0.0 if abs_err == 0 else float("inf"))
        rep.max_abs_err = max(rep.max_abs_err, abs_err)
        rep.max_rel_err = max(rep.max_rel_err, rel_err)
        if abs_err > atol + rtol * abs(fb):
            rep.mismatches += 1
            rep.passed = False
            if len(rep.detail) < 10:
                rep.detail.append(f"value {idx}: {ft!r} vs {fb!r} (abs {abs_err:.3e})")
    return rep


def run_tuning(evaluator: B200Evaluator, config: ga.GAConfig, out_dir=None,
               atol: float = DEFAULT_ATOL, rtol: float = DEFAULT_RTOL, echo=print) -> tuple:
    """Baseline, GA, verification and reports; returns (report document, verification ok)."""
    gene_len = evaluator.gene_length
    if hasattr(evaluator, "size"):
        what = (f"Himeno {evaluator.size.name} {evaluator.size.I}x{evaluator.size.J}x"
                f"{evaluator.size.K}, nn={evaluator.nn}")
    else:
        what = f"generated executor {evaluator.spec.name}"
    echo(f"gene length {gene_len}; evaluator: B200 x {evaluator.max_concurrency} worker slot(s), "
         f"{what}")
    t0 = time.perf_counter()
    baseline_s = measure_baseline(evaluator, gene_len)
    echo(f"baseline (all-CPU) time: {baseline_s:.6g} s")

    def on_generation(rec):
        echo(f"generation {rec.generation}: best so far {rec.best_time_s:.6g} s")

    result = ga.run_ga(config, gene_len, evaluator, on_generation)
    best = result.best
    ratio = baseline_s / best.time_s
    echo(f"best genome {ga.genome_str(best.genome)} time {best.time_s:.6g} s "
         f"ratio {ratio:.3f}x ({result.evaluations} evaluations)")
    if best.eval_source == "penalty" or best.timed_out:
        # every evaluated pattern failed or timed out: nothing ran to verify.  The
        # reference aborts here (run_for_output raises BaselineFailure, cli.py:265 /
        # evaluators.py:187); the run is reported, but as not passed (exit code 3)
        verification = {"status": "no-runnable-pattern",
                        "reason": f"best individual did not run: {best.diagnostic or 'timeout'}"}
        passed = False
        echo("verification: FAIL (no runnable pattern was evaluated)")
    else:
        base_out = evaluator.run_for_output((0,) * gene_len)
        tuned_out = evaluator.run_for_output(best.genome)
        diff = verify_results(base_out, tuned_out, atol, rtol)
        verification = diff.to_json() | {"status": "ran"}
        passed = diff.passed
        echo(f"verification: {'pass' if diff.passed else 'FAIL'} "
             f"(max abs err {diff.max_abs_err:.3e})")
    plan = evaluator.plan(best.genome)
    report = {
        "baseline_time_s": baseline_s,
        "best_time_s": best.time_s,
        "improvement_ratio": ratio,
        "best_genome": ga.genome_str(best.genome),
        "gene_length": gene_len,
        "kinds": {str(l): evaluator.kinds[l].value for l in evaluator.eligible_ids},
        "plan": plan.to_json(evaluator.refs),
        "verification": verification,
        "evaluations": result.evaluations,
        "ga": {"population": config.population, "generations": config.generations,
               "crossover_rate": config.crossover_rate, "mutation_rate": config.mutation_rate,
               "rng_seed": config.rng_seed},
        "note": "",
        "b200": {"best_run": evaluator.stats.get(best.genome, {}),
                 "worker_slots": evaluator.max_concurrency,
                 "transfer_mode": evaluator.transfer_mode,
                 "wall_s": time.perf_counter() - t0},
    }
    if out_dir is not None:
        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        (out / "report.json").write_text(json.dumps(report, indent=2, sort_keys=True) + "\n")
        with (out / "generations.jsonl").open("w") as fh:
            for rec in result.records:
                fh.write(json.dumps(rec.to_json(), sort_keys=True) + "\n")
        meta = {"written_at": time.strftime("%Y-%m-%dT%H:%M:%S%z"), "host": platform.node(),
                "python": platform.python_version()}
        (out / "meta.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    return report, passed


# device memory one B200 can give evaluator contexts (of ~180 GB; headroom for
# the runtime, the scratch rotation buffer and other tenants)
DEVICE_BYTES_FOR_CONTEXTS = 150e9
MAX_AUTO_WORKERS = 8


def auto_workers(size: str, n_dev: int, cpus: int) -> int:
    """`--workers-per-device auto`: host cores per GPU, capped so the contexts fit in
    device memory (each holds 15 pitched fields: L ~2 GB, XL ~16.3 GB) and in host
    pinned memory, and by a small constant (more concurrent runs than that only
    contend for the host cores and the PCIe link)."""
    from .apps import himeno
    sz = himeno.size(size)
    pitch = -(-(sz.K + 4) // 32) * 32
    per_ctx_dev = 15 * sz.I * sz.J * pitch * 4
    per_ctx_host = 14 * sz.I * sz.J * sz.K * 4
    by_cores = max(1, cpus // max(1, n_dev))
    by_mem = max(1, int(DEVICE_BYTES_FOR_CONTEXTS // per_ctx_dev))
    try:
        import os
        host_bytes = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        by_host = max(1, int(0.5 * host_bytes // (per_ctx_host * max(1, n_dev))))
    except (ValueError, OSError, AttributeError):
        by_host = MAX_AUTO_WORKERS
    return max(1, min(by_cores, by_mem, by_host, MAX_AUTO_WORKERS))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="GA offload search on B200s")
    ap.add_argument("--app", default=None,
                    help="a generated executor (generic.APPS, e.g. ft_s) instead of Himeno")
    ap.add_argument("--genes", default="verified", choices=["all", "verified", "screened"],
                    help="generated executors: the gene space (execution probe)")
    ap.add_argument("--size", default="M")
    ap.add_argument("--nn", type=int, default=3)
    ap.add_argument("--population", type=int, default=10)
    ap.add_argument("--generations", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--devices", default="0", help="comma list of GPU ids, or 'all'")
    ap.add_argument("--workers-per-device", default="1",
                    help="concurrent evaluations per GPU, or 'auto' (host cores / GPUs)")
    ap.add_argument("--transfer-mode", default="batched", choices=["batched", "per-loop"])
    ap.add_argument("--host-build", default="tuned", choices=["tuned", "reference"],
                    help="genes = 0: the library's tuned host loops, or the program's loops "
                         "built like the reference's compile template (gcc -O2)")
    ap.add_argument("--checkpoint", default=None,
                    help="JSONL of every fresh measurement (with its metrics); rerun with the "
                         "same file to resume an interrupted search (checkpoint.py)")
    ap.add_argument("--out")
    args = ap.parse_args(argv)
    devices = "all" if args.devices == "all" else [int(d) for d in args.devices.split(",")]
    if args.workers_per_device == "auto":
        import os
        from . import native
        n_dev = native.device_count() if devices == "all" else len(devices)
        workers = auto_workers(args.size, n_dev, os.cpu_count() or 1)
    else:
        workers = int(args.workers_per_device)
    cfg = ga.GAConfig(population=args.population, generations=args.generations,
                      rng_seed=args.seed)
    if args.app:
        from .generic import GenEvaluator
        from . import native
        devs = list(range(native.device_count())) if devices == "all" else devices
        with GenEvaluator(args.app, devices=devs, workers_per_device=workers,
                          transfer_mode=args.transfer_mode, nested_policy="outermost",
                          verify_each=args.genes != "all",
                          genes=None if args.genes == "all" else args.genes) as ev:
            _report, ok = run_tuning(ev, cfg, args.out)
        return 0 if ok else 3
    with B200Evaluator(args.size, nn=args.nn, devices=devices,
                       workers_per_device=workers,
                       transfer_mode=args.transfer_mode, host_build=args.host_build) as ev:
        plugin = ev
        if args.checkpoint:
            from .checkpoint import CheckpointedEvaluator
            plugin = CheckpointedEvaluator(ev, args.checkpoint)
        _report, ok = run_tuning(plugin, cfg, args.out)
        if args.checkpoint:
            print(f"checkpoint {args.checkpoint}: {plugin.measured} measured, "
                  f"{plugin.replayed} replayed")
    return 0 if ok else 3


if __name__ == "__main__":
    sys.exit(main())

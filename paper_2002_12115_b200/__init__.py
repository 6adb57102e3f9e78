"""B200-native GA fitness evaluation for GPU-offload pattern search (arXiv 2002.12115).

Hot path: genome -> transfer plan -> one execution of the application with
gene=1 loops as sm_100a kernels and gene=0 loops on the host -> measured time
-> GA.  Public surface mirrors the reference package ``acctuner``:

* ``ga``         fitness, GAConfig, init_population, roulette_pick, crossover,
                 mutate, EvalCache, evaluate_with_cache, run_ga
* ``plan``       Direction, PlanEntry, TransferPlan, Planner, plan_transfers,
                 compute_gpu_regions, hoist_and_batch, suppress_auto_transfers,
                 plan_for_genome
* ``evaluator``  MeasuredTime, B200Evaluator (the drop-in for ExternalEvaluator),
                 measure_baseline
* ``model``      structural program model (load/dump_structural)
* ``kinds``      DirectiveKind, eligible_ids, kind_map
* ``native``     ctypes binding of libhimeno_b200.so (C ABI include/himeno_b200.h)
"""

__version__ = "0.1.0"

#!/bin/bash
# One GPU round trip: tests, smoke, bench, launch list, one full ncu capture of the stencil.
# Usage (from the dev container): gpurun --timeout 1800 -- bash scripts/gpu_check.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-ga --no-cpu-baseline --no-other-grids --e2e-steps 1 > $OUT/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 5 -c 2 \
  -o $OUT/stencil python bench.py --steps 1 --warmup 3 --no-ga --no-cpu-baseline --no-other-grids --e2e-steps 1 > $OUT/ncu_full.log 2>&1
ls -la $OUT
tail -5 $OUT/pytest_gpu.log $OUT/smoke.log $OUT/bench.err
cat $OUT/bench.json $OUT/bench_ref.json

#!/bin/bash
# One GPU iteration: parity tests, a bench line, and an ncu launch list.
# usage (under gpurun): bash tools/gpu_cycle.sh TAG
TAG=${1:-x}
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_$TAG.log
python bench.py --no-oracle --no-e2e > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-oracle --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_$TAG.log 2>&1; echo "launches rc=$?"

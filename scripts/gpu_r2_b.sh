#!/bin/bash
# Dev: GPU tests (all, no -x) + c5b/c5/c4 bench lines + c5b launch list.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for c in c5b c5 c4; do
  timeout 600 python bench.py --config $c --no-configs --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv \
    python bench.py --config c5b --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2> gpurun_out/launches_c5b.err
ls -la gpurun_out

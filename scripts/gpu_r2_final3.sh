#!/bin/bash
# Round-2 closing evidence: default bench line (all configs), reference arm, launch lists of c4 and c5b.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2h_bench_default.json 2> gpurun_out/r2h_bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2h_bench_reference.json 2>&1
for c in c4 c5b; do
  st=8; [ $c = c5b ] && st=2
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_$c.csv \
      python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
done
ls -la gpurun_out | tail -6

#!/bin/bash
# Round-2 final evidence pass (session 3): the default bench line, the reference arm, c5b's launch
# list with the saved-chunk backward, the full GPU test suite and compute-sanitizer.  Into gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r2f_gputest.log 2>&1; echo "tests exit $?" >> gpurun_out/r2f_gputest.log
timeout 900 python bench.py > gpurun_out/r2f_bench_default.json 2> gpurun_out/r2f_bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_bench_reference.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches_c5b.csv \
    python bench.py --config c5b --steps 2 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
for t in memcheck racecheck synccheck; do
  echo "## $t" >> gpurun_out/r2f_sanitizer.txt
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize_smoke.py 2>&1 | tail -4 >> gpurun_out/r2f_sanitizer.txt
done
ls -la gpurun_out

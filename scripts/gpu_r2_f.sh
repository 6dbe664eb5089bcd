#!/bin/bash
set -u
mkdir -p gpurun_out
python scripts/c1_graph.py paper_2001_00706_b200/libsig.so paper_2001_00706_b200/libsig_lc4.so paper_2001_00706_b200/libsig_lc8.so > gpurun_out/c1_graph.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_f.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_f.txt
for c in c5 c5b c1; do
timeout 600 python bench.py --config $c --no-configs --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv \
    python bench.py --config c5b --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2> gpurun_out/launches_c5b.err
ls -la gpurun_out

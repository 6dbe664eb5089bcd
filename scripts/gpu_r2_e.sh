#!/bin/bash
set -u
mkdir -p gpurun_out
python scripts/c1_graph.py paper_2001_00706_b200/libsig.so paper_2001_00706_b200/libsig_lc2.so paper_2001_00706_b200/libsig_lc4.so paper_2001_00706_b200/libsig_lc8.so > gpurun_out/c1_graph.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_e.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_e.txt
timeout 600 python bench.py --config c5b --no-configs --no-cpu-baseline > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv \
    python bench.py --config c5b --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2> gpurun_out/launches_c5b.err
for b in 512 256 128; do
  timeout 600 python bench.py --batch $b --no-configs --no-cpu-baseline --steps 100 > gpurun_out/bench_c2_b$b.json 2> gpurun_out/bench_c2_b$b.err
done
ls -la gpurun_out

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_logsig_combine.py -m gpu -q -rf -s -k "many_rows or rows_kernel or stream" > gpurun_out/pytest_gpu_j.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_j.txt
timeout 600 python bench.py --config c3l --no-configs --no-cpu-baseline --steps 50 > gpurun_out/bench_c3l.json 2> gpurun_out/bench_c3l.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3l.csv \
    python bench.py --config c3l --steps 3 --warmup 2 --no-cpu-baseline --no-configs > /dev/null 2>&1

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_logsig_combine.py -m gpu -q -rf -s -k "many_rows or rows_kernel or stream" > gpurun_out/pytest_gpu_k.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_k.txt
timeout 600 python bench.py --config c3l --no-configs --no-cpu-baseline --steps 50 > gpurun_out/bench_c3l.json 2> gpurun_out/bench_c3l.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:logsig_rows -s 1 -c 1 -o /tmp/c3l_rows \
    python bench.py --config c3l --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/c3l_rows.ncu-rep > gpurun_out/c3l_rows_ncu.txt 2>&1

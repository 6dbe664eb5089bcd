#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd_chunked.py tests/test_gpu_signature.py tests/test_gpu_dist.py -m gpu -q -rf -s -k "chunk or c5 or long or dist or backward" > gpurun_out/pytest_gpu_c.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_c.txt
timeout 600 python bench.py --config c5b --no-configs --no-cpu-baseline > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv \
    python bench.py --config c5b --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2> gpurun_out/launches_c5b.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sig_bwd_kernel -s 1 -c 1 -o gpurun_out/c5b_k2_full \
    python scripts/profile_c2.py c5b 2 > /dev/null 2> gpurun_out/c5b_k2_full.err
ls -la gpurun_out

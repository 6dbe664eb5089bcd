#!/bin/bash
# Dev: round-2 first evidence pass (GPU tests, default bench line with configs block, c2 launch list,
# full capture of c2's K2).  Everything lands in gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2> gpurun_out/launches_c2.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sig_bwd2p_kernel -s 1 -c 1 -o gpurun_out/c2_k2p_full \
    python scripts/profile_c2.py c2 3 > /dev/null 2> gpurun_out/c2_k2p_full.err
ls -la gpurun_out

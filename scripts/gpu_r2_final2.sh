#!/bin/bash
# Round-2 final evidence refresh after the grouped-chunk plan change: default bench line, c5 launch list.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2g_bench_default.json 2> gpurun_out/r2g_bench_default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches_c5.csv \
    python bench.py --config c5 --steps 8 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sig_fwd_kernel -s 2 -c 1 -o /tmp/r2g_c5_k1 \
    python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/r2g_c5_k1.ncu-rep > gpurun_out/r2g_c5_k1_ncu.txt 2>&1
ncu -i /tmp/r2g_c5_k1.ncu-rep --page source --csv --print-source sass > /tmp/r2g_sass.csv 2>/dev/null
python scripts/sass_opmix.py /tmp/r2g_sass.csv >> gpurun_out/r2g_c5_k1_ncu.txt 2>&1
ls -la gpurun_out | tail -5

#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd_chunked.py tests/test_gpu_signature.py tests/test_gpu_dist.py -m gpu -q -rf -s -k "chunk or c5 or long or dist" > gpurun_out/pytest_gpu_d.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_d.txt
timeout 600 python bench.py --config c5b --no-configs --no-cpu-baseline > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv \
    python bench.py --config c5b --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2> gpurun_out/launches_c5b.err
for b in 1024 512 256 128; do
  timeout 600 python bench.py --batch $b --no-configs --no-cpu-baseline --steps 100 > gpurun_out/bench_c2_b$b.json 2> gpurun_out/bench_c2_b$b.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_b128.csv \
    python bench.py --batch 128 --steps 4 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv \
    python bench.py --config c1 --steps 20 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sig_fwd -s 3 -c 1 -o gpurun_out/c1_k1_full \
    python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
ls -la gpurun_out

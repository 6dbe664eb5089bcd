#!/bin/bash
# Dev: bench lines for every BASELINE config + launch lists + full captures, into gpurun_out/.
set -u
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do
  python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv \
    python bench.py --config c4 --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sig_bwd2_kernel -s 1 -c 1 -o gpurun_out/c2_k2_full \
    python scripts/profile_c2.py c2 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sig_fwd2_kernel -s 1 -c 1 -o gpurun_out/c2_k1_full \
    python scripts/profile_c2.py c2 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sig_fwd_stream_kernel -s 1 -c 1 -o gpurun_out/c3_stream_full \
    python scripts/profile_c2.py c3 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sig_bwd_kernel -s 1 -c 1 -o gpurun_out/c4_k2_full \
    python scripts/profile_c2.py c4 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sig_fwd_kernel -s 1 -c 1 -o gpurun_out/c5_k1_full \
    python scripts/profile_c2.py c5 3 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --config c5 --steps 8 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out

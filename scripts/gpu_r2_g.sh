#!/bin/bash
set -u
mkdir -p gpurun_out
python scripts/c1_graph.py paper_2001_00706_b200/libsig.so paper_2001_00706_b200/libsig_lc4.so paper_2001_00706_b200/libsig_lc8.so paper_2001_00706_b200/libsig_lc32.so > gpurun_out/c1_graph.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu_g.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_g.txt
for c in c5 c1; do
timeout 600 python bench.py --config $c --no-configs --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sig_fwd -s 3 -c 1 -o gpurun_out/c1_k1_full \
    python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-configs > /dev/null 2>&1
ls -la gpurun_out

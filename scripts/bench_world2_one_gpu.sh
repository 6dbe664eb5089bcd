#!/bin/bash
# Dev: the N-rank path of bench.py on ONE GPU (all ranks on cuda:0, gloo): does every arm run and
# print one line with n_gpus = 2?  Numbers are not multi-GPU measurements.
set -u
mkdir -p gpurun_out
export SIGB200_BENCH_SHARE_GPU=1
timeout 900 python bench.py --gpus 2 --backend gloo --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/n2_default.json 2> gpurun_out/n2_default.err
timeout 600 python bench.py --gpus 2 --backend gloo --scaling strong --steps 20 --warmup 3 --no-configs > gpurun_out/n2_strong.json 2> gpurun_out/n2_strong.err
timeout 600 python bench.py --gpus 2 --backend gloo --config c5b --steps 3 --warmup 3 --no-configs > gpurun_out/n2_c5b.json 2> gpurun_out/n2_c5b.err
timeout 600 python bench.py --gpus 2 --backend gloo --config c4 --steps 10 --warmup 3 --no-configs > gpurun_out/n2_c4.json 2> gpurun_out/n2_c4.err
timeout 600 python bench.py --gpus 2 --impl reference --steps 2 --warmup 3 > gpurun_out/n2_ref.json 2> gpurun_out/n2_ref.err

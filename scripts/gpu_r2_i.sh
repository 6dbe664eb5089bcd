#!/bin/bash
set -u
mkdir -p gpurun_out
L=paper_2001_00706_b200
python scripts/c5_time.py $L/libsig.so $L/libsig_nocontig.so > gpurun_out/c5_time.txt 2>&1
python scripts/c1_graph.py $L/libsig.so $L/libsig_nocontig.so > gpurun_out/c1_graph.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_signature.py tests/test_gpu_options.py tests/test_gpu_path.py -m gpu -q -rf > gpurun_out/pytest_gpu_i.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_i.txt

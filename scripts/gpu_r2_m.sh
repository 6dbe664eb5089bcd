#!/bin/bash
set -u
mkdir -p gpurun_out
L=paper_2001_00706_b200
python scripts/c4_time.py $L/libsig.so $L/libsig_pb5.so $L/libsig.so $L/libsig_pb5.so > gpurun_out/c4_time.txt 2>&1
SIGB200_LIB=$PWD/$L/libsig_pb5.so timeout 900 python -m pytest tests/test_gpu_logsig_combine.py tests/test_gpu_signature.py -m gpu -q -rf -k "c4 or 4-7 or backward" > gpurun_out/pytest_gpu_m.txt 2>&1; echo "pytest pb5 rc=$?" >> gpurun_out/pytest_gpu_m.txt

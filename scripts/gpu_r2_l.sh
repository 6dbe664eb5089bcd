#!/bin/bash
set -u
mkdir -p gpurun_out
L=paper_2001_00706_b200
python scripts/c3l_time.py $L/libsig.so $L/libsig_db.so $L/libsig.so $L/libsig_db.so > gpurun_out/c3l_time.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_logsig_combine.py -m gpu -q -rf -k "many_rows or rows_kernel or stream" > gpurun_out/pytest_gpu_l.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_l.txt
SIGB200_LIB=$PWD/$L/libsig_db.so timeout 900 python -m pytest tests/test_gpu_logsig_combine.py -m gpu -q -rf -k "many_rows or rows_kernel" >> gpurun_out/pytest_gpu_l.txt 2>&1; echo "pytest db rc=$?" >> gpurun_out/pytest_gpu_l.txt

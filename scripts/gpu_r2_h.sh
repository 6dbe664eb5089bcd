#!/bin/bash
set -u
mkdir -p gpurun_out
L=paper_2001_00706_b200
python scripts/c5_time.py $L/libsig.so $L/libsig_nocontig.so $L/libsig.so $L/libsig_nocontig.so > gpurun_out/c5_time.txt 2>&1
python scripts/c1_graph.py $L/libsig.so $L/libsig_nocontig.so > gpurun_out/c1_graph.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sig_fwd_kernel -s 2 -c 1 -o gpurun_out/c5_k1_contig \
    python scripts/profile_c2.py c5 3 > /dev/null 2>&1
SIGB200_LIB=$PWD/$L/libsig_nocontig.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:sig_fwd_kernel -s 2 -c 1 -o gpurun_out/c5_k1_nocontig \
    python scripts/profile_c2.py c5 3 > /dev/null 2>&1
ls -la gpurun_out

#!/bin/bash
# Round-2 evidence pass (python scripts, not the driver's run): bench lines (default c2 + configs block, reference arm), launch lists of
# every config, --set full captures of the dominant kernels, compute-sanitizer.  Into gpurun_out/.
set -u
mkdir -p gpurun_out
B="--no-cpu-baseline --no-configs"
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_reference.json 2>&1
for c in c2 c4 c5 c5b c1 c3 c3l; do
  st=8; [ $c = c5b ] && st=2; [ $c = c1 ] && st=20
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$c.csv \
      python bench.py --config $c --steps $st --warmup 3 $B > /dev/null 2>&1
done
# each capture is summarised on the box (the reports themselves exceed gpurun's 64 MiB pull limit)
capb() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-1} -c 1 -o /tmp/r2_$1 \
          python bench.py --config $3 --steps 2 --warmup 1 --no-cpu-baseline --no-configs > /dev/null 2>&1
        python scripts/ncu_summary.py /tmp/r2_$1.ncu-rep > gpurun_out/r2_$1_ncu.txt 2>&1
        ncu -i /tmp/r2_$1.ncu-rep --page source --csv --print-source sass > /tmp/r2_$1_sass.csv 2>/dev/null
        python scripts/sass_opmix.py /tmp/r2_$1_sass.csv >> gpurun_out/r2_$1_ncu.txt 2>&1; }
cap() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${4:-1} -c 1 -o /tmp/r2_$1 \
          python scripts/profile_c2.py $3 3 > /dev/null 2>&1
        python scripts/ncu_summary.py /tmp/r2_$1.ncu-rep > gpurun_out/r2_$1_ncu.txt 2>&1
        ncu -i /tmp/r2_$1.ncu-rep --page source --csv --print-source sass > /tmp/r2_$1_sass.csv 2>/dev/null
        python scripts/sass_opmix.py /tmp/r2_$1_sass.csv >> gpurun_out/r2_$1_ncu.txt 2>&1; }
cap c2_k1 sig_fwd2_kernel c2
cap c2_k2 sig_bwd2p_kernel c2
cap c4_k2 sig_bwd_kernel c4
cap c4_k5 logsig_bwd c4
cap c4_k1 sig_fwd2_kernel c4
cap c5_k1 sig_fwd_kernel c5 2
cap c3_stream sig_fwd_stream_kernel c3
cap c5b_scan scan_group_t c5b 2
cap c5b_k2 sig_bwd_kernel c5b 1
capb c3l_k4 logsig_rows c3l 1
capb c1_k1 sig_fwd c1 3
for t in memcheck racecheck synccheck; do
  echo "## $t" >> gpurun_out/r2_sanitizer.txt
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize_smoke.py 2>&1 | tail -4 >> gpurun_out/r2_sanitizer.txt
done
ls -la gpurun_out

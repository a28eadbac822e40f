#!/bin/bash
# Round-2 ncu captures (run under gpurun, one GPU): side-task kernels INSIDE a
# harvest (scripts/ncu_harvest.py brackets the timed run with
# cudaProfilerStart/Stop) and the tensor-pipe utilisation of the stand-in
# GEMMs that define the bubbles.
set -u
out=gpurun_out
export FR_HARNESS_NO_PROFILE_GATE=1
NCU="ncu --clock-control none --profile-from-start off"
# 1. launch list of one harvest window (names + device time)
$NCU --metrics gpu__time_duration.sum --csv --log-file $out/r2_harvest_launches.csv \
  python scripts/ncu_harvest.py image > $out/r2_ncu_list.log 2>&1
gemm=$(grep -v -E 'img_|pr_|sgd_|gap_kernel|link_|stamp_|ID' $out/r2_harvest_launches.csv | awk -F'","' 'NR>1{print $5}' | sort | uniq -c | sort -rn | head -1 | awk '{print $2}')
echo "gemm kernel: $gemm" >> $out/r2_ncu_list.log
# 2. K5 in the harvest: all SMs and a 20-SM budget
$NCU --set full --import-source on -k regex:img_resize2x -s 6 -c 1 -o $out/r2_k5_harvest \
  python scripts/ncu_harvest.py image > $out/r2_ncu_k5.log 2>&1
$NCU --set full --import-source on -k regex:img_resize2x -s 6 -c 1 -o $out/r2_k5_harvest_20sm \
  python scripts/ncu_harvest.py image 20 > $out/r2_ncu_k5_20.log 2>&1
# 3. PageRank and Graph-SGD in the harvest
$NCU --set full --import-source on -k regex:pr_pull -s 4 -c 1 -o $out/r2_pr_harvest \
  python scripts/ncu_harvest.py pagerank > $out/r2_ncu_pr.log 2>&1
$NCU --set full --import-source on -k regex:sgd_user -s 4 -c 1 -o $out/r2_sgd_harvest \
  python scripts/ncu_harvest.py sgd > $out/r2_ncu_sgd.log 2>&1
# 4. the stand-in GEMM: tensor pipe
gemm=${gemm%%[(<]*}
if [ -n "$gemm" ]; then
  $NCU --set full -k "regex:^${gemm}" -s 4 -c 2 -o $out/r2_gemm_harvest \
    python scripts/ncu_harvest.py image > $out/r2_ncu_gemm.log 2>&1
fi
ls -la $out/r2_*.ncu-rep

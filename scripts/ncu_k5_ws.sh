#!/bin/bash
# ncu of the warp-specialised K5 (img_resize2x_wm_ws): standalone 16-frame
# launches on all SMs and on a 16-SM budget (cold, serialised), and inside a
# harvest on a 12-SM budget (the controller's operating point).
set -u
out=gpurun_out
NCU="ncu --clock-control none"
$NCU --set full --import-source on -k regex:img_resize2x -s 8 -c 1 -o $out/r2s_k5ws_148 \
  python scripts/img_microbench.py 16 2 > $out/r2s_ncu_k5ws_148.log 2>&1
FR_IMG_MAX_SMS=16 $NCU --set full --import-source on -k regex:img_resize2x -s 8 -c 1 -o $out/r2s_k5ws_16 \
  python scripts/img_microbench.py 16 2 > $out/r2s_ncu_k5ws_16.log 2>&1
FR_HARNESS_NO_PROFILE_GATE=1 $NCU --profile-from-start off --set full --import-source on -k regex:img_resize2x -s 6 -c 1 \
  -o $out/r2s_k5ws_harvest_12 python scripts/ncu_harvest.py image 12 > $out/r2s_ncu_k5ws_h12.log 2>&1
ls -la $out/r2s_k5ws*.ncu-rep

#!/bin/bash
# Round-2 session-3 ncu captures (one GPU, under gpurun): the harvest window's
# launch list and the warp-specialised K5 inside a harvest, on all SMs and on
# an 8-SM-equivalent budget (the controller's operating point).
set -u
out=gpurun_out
export FR_HARNESS_NO_PROFILE_GATE=1
NCU="ncu --clock-control none --profile-from-start off"
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file $out/r2s_harvest_launches.csv python scripts/ncu_harvest.py image 8 > $out/r2s_ncu_list.log 2>&1
$NCU --set full --import-source on -k regex:img_resize2x -s 6 -c 1 -o $out/r2s_k5ws_harvest_all \
  python scripts/ncu_harvest.py image > $out/r2s_ncu_k5h_all.log 2>&1
$NCU --set full --import-source on -k regex:img_resize2x -s 6 -c 1 -o $out/r2s_k5ws_harvest_8 \
  python scripts/ncu_harvest.py image 8 > $out/r2s_ncu_k5h_8.log 2>&1
ls -la $out/r2s_k5ws_harvest_*.ncu-rep $out/r2s_harvest_launches.csv

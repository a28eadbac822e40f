#!/bin/bash
# A/B of the K5 variants at several SM budgets; standalone, device-timed
# (scripts/img_microbench.py, 16-frame steps).  Variants:
#   ws    warp-decoupled kernel, dp4a math (the default)
#   bar1  per-row-barrier kernel, dp4a math (FR_IMG_CFG=bar)
#   bar0  per-row-barrier kernel, 16-bit lane math (FR_IMG_MATH=0, round 1)
for sms in ${SMS:-5 8 16 148}; do
  echo "ws   sms=$sms $(FR_IMG_MAX_SMS=$sms python scripts/img_microbench.py 16 20)"
  echo "bar1 sms=$sms $(FR_IMG_CFG=bar FR_IMG_MAX_SMS=$sms python scripts/img_microbench.py 16 20)"
  [ -n "$BAR0" ] && echo "bar0 sms=$sms $(FR_IMG_MATH=0 FR_IMG_MAX_SMS=$sms python scripts/img_microbench.py 16 20)"
done

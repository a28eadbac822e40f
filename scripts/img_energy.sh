#!/bin/bash
# K5 energy per pixel across kernel variants and SM budgets (scripts/img_energy.py)
for sms in 8 16 48 148; do
  FR_IMG_MAX_SMS=$sms python scripts/img_energy.py 3
  FR_IMG_PIPES=3 FR_IMG_MAX_SMS=$sms python scripts/img_energy.py 3
  FR_IMG_CFG=bar FR_IMG_MAX_SMS=$sms python scripts/img_energy.py 3
  FR_IMG_MATH=0 FR_IMG_MAX_SMS=$sms python scripts/img_energy.py 3
done

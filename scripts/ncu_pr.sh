#!/bin/bash
# ncu of the PageRank pull kernel: standalone (scripts/pr_microbench.py), with
# the source page (instructions executed per SASS line) for the instruction diet
set -u
out=gpurun_out
ncu --clock-control none --set full --import-source on -k regex:pr_pull -s 6 -c 1 -o $out/r2s_pr \
  python scripts/pr_microbench.py > $out/r2s_ncu_pr.log 2>&1
ls -la $out/r2s_pr.ncu-rep

#!/bin/bash
# A/B of two builds of the library on one box: scratch/ab/A.so and scratch/ab/B.so, alternating.
# usage: scratch/ab.sh [rounds] [stage_times args...]
R=${1:-2}; shift
for r in $(seq $R); do
  for v in A B; do
    cp scratch/ab/$v.so paper_2501_12369_b200/libdarbs_cuda.so
    echo "== $v (round $r)"
    python scratch/stage_times.py "$@" 2>&1 | grep -o "^[a-z-]* \|'render_fwd': [0-9.]*\|'render_bwd': [0-9.]*\|'cull': [0-9.]*\|'binning': [0-9.]*\|'loss': [0-9.]*\|total [0-9.]*" | paste -sd' ' | sed 's/ \([a-z-]* \) /\n\1/g'
  done
done

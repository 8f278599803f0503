#!/bin/bash
V=$1; shift
for r in 1 2; do for v in $V; do
  cp scratch/ab/$v.so paper_2501_12369_b200/libdarbs_cuda.so
  echo "== $v (round $r)"; python scratch/stage_times.py "$@" 2>&1 | grep -o "^[a-z-]* \|'render_fwd': [0-9.]*\|total [0-9.]*" | paste - - -
done; done

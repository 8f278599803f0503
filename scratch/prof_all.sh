#!/bin/bash
# ncu captures of one training iteration per DARBF kernel (run under gpurun): a launch list and a
# --set full capture, summarised ON the box (the reports are ~50 MB each; only the markdown and the
# launch CSVs travel back).
mkdir -p gpurun_out
for k in "$@"; do
  ncu --metrics gpu__time_duration.sum --clock-control none -s 90 -c 64 --csv --log-file gpurun_out/launches_r1_$k.csv python scratch/prof_step.py $k > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -s 90 -c 34 -o /tmp/step_r1_$k -f python scratch/prof_step.py $k > /dev/null 2>&1
  python scratch/make_profile_summary.py /tmp/step_r1_$k.ncu-rep gpurun_out/r1_training_step_$k.md "Round 1 - one training iteration (scene B of bench.py: 1 M primitives, 1920x1080, $k preset, L1 + D-SSIM loss), kernels of the hot path" "darbs_b200"
  rm -f /tmp/step_r1_$k.ncu-rep
done
ls -la gpurun_out/*.md gpurun_out/launches_r1_*.csv

#!/bin/bash
# ncu captures of one training iteration per DARBF kernel (run under gpurun): a launch list and a
# --set full capture, summarised ON the box (the reports are ~50 MB each; only the markdown and the
# launch CSVs travel back).   usage: scratch/prof_all.sh <round tag, e.g. r2> kernel...
R=$1; shift
mkdir -p gpurun_out
for k in "$@"; do
  ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 48 --csv --log-file gpurun_out/launches_${R}_$k.csv python scratch/prof_step.py $k > /dev/null 2>&1
  python scratch/launch_list.py gpurun_out/launches_${R}_$k.csv gpurun_out/${R}_launches_$k.md "Round ${R#r} - launch list of one training iteration ($k, scene B, 1 M primitives, 1080p, L1 + D-SSIM loss): ncu --metrics gpu__time_duration.sum --clock-control none over scratch/prof_step.py $k" project_kernel
  ncu --set full --clock-control none --import-source on -s 60 -c 24 -o /tmp/step_${R}_$k -f python scratch/prof_step.py $k > /dev/null 2>&1
  python scratch/make_profile_summary.py /tmp/step_${R}_$k.ncu-rep gpurun_out/${R}_training_step_$k.md "Round ${R#r} - one training iteration (scene B of bench.py: 1 M primitives, 1920x1080, $k preset, L1 + D-SSIM loss), kernels of the hot path" "darbs_b200"
  python scratch/traffic_json.py /tmp/step_${R}_$k.ncu-rep $k >> gpurun_out/${R}_traffic.jsonl
  rm -f /tmp/step_${R}_$k.ncu-rep
done
ls -la gpurun_out/*.md gpurun_out/launches_${R}_*.csv

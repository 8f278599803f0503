set -e
cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none -k regex:onesweep --launch-skip 40 --launch-count 1 -o gpurun_out/r2_sort scratch/sort/sort_bench_512_16_8 > gpurun_out/r2_sort_ncu.log 2>&1 || true
ncu -i gpurun_out/r2_sort.ncu-rep --page raw --csv > gpurun_out/r2_sort_raw.csv 2>/dev/null || true
tail -3 gpurun_out/r2_sort_ncu.log

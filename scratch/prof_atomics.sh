#!/bin/bash
# L2-level atomic / reduction counters of the kernels that issue red.global / atom.global (run under gpurun).
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,smsp__inst_executed_op_global_red.sum,smsp__inst_executed_op_global_atom.sum,smsp__inst_executed_op_shared_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,dram__bytes_read.sum,dram__bytes_write.sum
for k in "$@"; do
  ncu --metrics $M --clock-control none -k regex:"render_bwd|expand_kernel|onesweep|depth_histogram|project_kernel|cull_kernel|render_fwd" -s 20 -c 14 --csv --log-file gpurun_out/r2_atomics_$k.csv python scratch/prof_step.py $k > /dev/null 2>&1
done
ls -la gpurun_out/r2_atomics_*.csv

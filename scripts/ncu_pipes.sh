#!/bin/bash
# Pipe utilisation + per-instruction stalls of the encoder (1 GPU); keeps copies under /tmp on the box too.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2604_17172_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
B=${NCU_BYTES:-1073741824}
M="sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.per_cycle_active"
for k in ${NCU_KERNELS:-k_fused}; do
  ncu --metrics $M --clock-control none -k regex:$k -s 1 -c 1 --csv \
    python bench.py --steps 1 --warmup 1 --bytes $B --no-cpu-baseline --no-e2e --no-loopback > gpurun_out/pipes_$k.csv 2> gpurun_out/pipes_$k.err
done

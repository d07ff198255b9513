#!/bin/bash
# ncu captures of the codec kernels (1 GPU): launch list + one full-set capture per kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=${NCU_BYTES:-1073741824}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --bytes $B --no-cpu-baseline --no-e2e --no-loopback --no-dtypes --no-c1 > gpurun_out/ncu_launch_bench.log 2>&1
for k in ${NCU_KERNELS:-k_fused k_decode k_hist}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k -f \
    python bench.py --steps 1 --warmup 1 --bytes $B --no-cpu-baseline --no-e2e --no-loopback --no-dtypes --no-c1 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out/

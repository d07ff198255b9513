#!/bin/bash
# Per-instruction view of the codec kernels (1 GPU): one full-set capture each with source
# correlation, exported as SASS-level CSV (inst_executed + warp stall samples per instruction).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2604_17172_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
B=${NCU_BYTES:-1073741824}
for k in ${NCU_KERNELS:-k_fused k_decode}; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/src_$k -f \
    python bench.py --steps 1 --warmup 1 --bytes $B --no-cpu-baseline --no-e2e --no-loopback > gpurun_out/ncu_src_$k.log 2>&1
  ncu -i gpurun_out/src_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$k.csv 2>&1
  ncu -i gpurun_out/src_$k.ncu-rep --page raw --csv > gpurun_out/raw_$k.csv 2>&1
done
ls -la gpurun_out/

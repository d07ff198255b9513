#!/bin/bash
# A/B ncu --set full captures of one kernel across libuzip variants (default + variants/*.so).
#   NCU_KERNEL=k_fused VARIANTS="v1 g8" ./scripts/ncu_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${NCU_KERNEL:-k_fused}
B=${NCU_BYTES:-1073741824}
for v in default ${VARIANTS}; do
  if [ "$v" = default ]; then L=""; else L="$PWD/paper_2604_17172_b200/variants/$v.so"; fi
  UZIP_LIB_PATH=$L ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/ab_${K}_$v -f \
    python bench.py --steps 1 --warmup 1 --bytes $B --no-cpu-baseline --no-e2e --no-loopback --no-dtypes --no-c1 > gpurun_out/ab_${K}_$v.log 2>&1
  echo "$v rc=$?"
done

#!/bin/bash
# Round-2 measurement on 1 GPU: default bench line, reference arm, smoke, ncu launch list of the bench
# command, full-set captures of k_fused and k_decode (1 GiB), pipe utilisation of k_fused.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2604_17172_b200 import _build; _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 600 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
NCU_KERNELS="k_fused k_decode" ./scripts/ncu_codec.sh > /dev/null 2>&1
NCU_KERNELS="k_fused" ./scripts/ncu_pipes.sh > /dev/null 2>&1
cat gpurun_out/bench_default.log gpurun_out/bench_reference.log gpurun_out/smoke.log

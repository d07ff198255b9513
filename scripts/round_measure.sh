#!/bin/bash
# Round measurement on 1 GPU: default bench line, ncu launch list of the same command, full-set captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2604_17172_b200 import _build; print(_build.build())" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 600 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
./scripts/ncu_codec.sh
cat gpurun_out/bench_default.log gpurun_out/bench_reference.log gpurun_out/smoke.log
timeout 600 python scripts/ablations.py --out gpurun_out/ablations.json > gpurun_out/ablations.log 2>&1
tail -1 gpurun_out/ablations.log

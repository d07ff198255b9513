#!/bin/bash
# One gpurun call: GPU tests (per-test timeout, durations), then a short bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "from paper_2604_17172_b200 import _build; print(_build.build())" > gpurun_out/build.log 2>&1
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q -x --timeout 240 --durations=25 ${PYTEST_ARGS} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py $BENCH > gpurun_out/bench.log 2>&1
  echo "bench rc=$?" >> gpurun_out/bench.log
fi
tail -40 gpurun_out/gpu_tests.log
tail -5 gpurun_out/bench.log 2>/dev/null || true

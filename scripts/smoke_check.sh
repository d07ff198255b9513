#!/bin/bash
# smoke() plain, under CUDA_LAUNCH_BLOCKING=1, and under ncu (the driver's launch-list capture).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/smoke_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/smoke_plain.log
CUDA_LAUNCH_BLOCKING=1 python __graft_entry__.py > gpurun_out/smoke_blocking.log 2>&1; echo "blocking rc=$?" >> gpurun_out/smoke_blocking.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches.csv \
  python -c "import os; print('INJ', os.environ.get('CUDA_INJECTION64_PATH')); import __graft_entry__ as g; g.smoke()" \
  > gpurun_out/smoke_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/smoke_ncu.log
tail -n 3 gpurun_out/smoke_plain.log gpurun_out/smoke_blocking.log gpurun_out/smoke_ncu.log

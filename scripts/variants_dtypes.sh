#!/bin/bash
# Per-dtype (U[-1,1]) round-trip GB/s and the 1 GiB bf16 codec times of libuzip variants vs default.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2604_17172_b200 import _build; _build.build()" > /dev/null 2>&1
for v in default paper_2604_17172_b200/variants/*.so; do
  if [ "$v" = default ]; then L=""; else L="$PWD/$v"; fi
  UZIP_LIB_PATH=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-loopback --no-c1 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$v', d['encode']['ms'], d['decode']['ms'], {k: v['roundtrip_GBps'] for k, v in d['per_dtype_uniform'].items()})"
done

#!/bin/bash
# C1 (4 MiB) and 1 GiB codec timings of libuzip variants (paper_2604_17172_b200/variants/*.so) vs default.
cd "$(dirname "$0")/.."
python -c "from paper_2604_17172_b200 import _build; _build.build()" > /dev/null 2>&1
for v in default paper_2604_17172_b200/variants/*.so; do
  if [ "$v" = default ]; then L=""; else L="$PWD/$v"; fi
  UZIP_LIB_PATH=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-loopback --no-dtypes 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$(basename $v)', d['encode']['ms'], d['decode']['ms'], d['c1_4mib']['compress_us'], d['c1_4mib']['decompress_us'])"
done

#!/bin/bash
# C1 (4 MiB bf16) device time per compress / decompress call for libuzip variants (variants/*.so) vs default.
cd "$(dirname "$0")/.."
python -c "from paper_2604_17172_b200 import _build; _build.build()" > /dev/null 2>&1
for v in default paper_2604_17172_b200/variants/*.so; do
  if [ "$v" = default ]; then L=""; else L="$PWD/$v"; fi
  echo "$(basename $v)"; UZIP_LIB_PATH=$L python scripts/c1_host.py
done

#!/bin/bash
# Receiver-side (D item) and sender-side (E item) device times of a 1 GiB bf16 W P2P (scripts/p2p_sides.py)
# for the default library and every variant.
cd "$(dirname "$0")/.."
python -c "from paper_2604_17172_b200 import _build; _build.build()" > /dev/null 2>&1
for v in default paper_2604_17172_b200/variants/*.so; do
  if [ "$v" = default ]; then L=""; else L="$PWD/$v"; fi
  echo "== $v"; UZIP_LIB_PATH=$L timeout 300 python scripts/p2p_sides.py 2>&1 | tail -3
done

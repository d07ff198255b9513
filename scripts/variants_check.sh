#!/bin/bash
# A/B of libuzip variants on the 1 GiB codec bench (scripts/variants.sh), then each variant's codec parity tests.
cd "$(dirname "$0")/.."
./scripts/variants.sh
for v in paper_2604_17172_b200/variants/*.so; do
  echo "== parity $v"; UZIP_LIB_PATH=$PWD/$v timeout 600 python -m pytest tests/test_gpu_codec.py -q -x -m gpu 2>&1 | tail -1
done

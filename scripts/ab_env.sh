#!/bin/bash
# A/B of environment knobs on the N=1 bench: ENVS="A=1 B=2" -> one line per setting (plus default).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "from paper_2604_17172_b200 import _build; _build.build()" > /dev/null 2>&1
for e in default ${ENVS}; do
  for rep in 1 2; do
    if [ "$e" = default ]; then E=""; else E="$e"; fi
    env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-loopback --no-dtypes 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$e', d['encode']['ms'], d['decode']['ms'], d['value'], d['c1_4mib']['compress_us'], d['c1_4mib']['decompress_us'])"
  done
done

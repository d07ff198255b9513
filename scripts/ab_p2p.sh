#!/bin/bash
# loopback P2P (bench.py's context field) under env settings: ENVS="A=1 B=0"
cd "$(dirname "$0")/.."
python -c "from paper_2604_17172_b200 import _build; _build.build()" > /dev/null 2>&1
for e in default ${ENVS}; do
  if [ "$e" = default ]; then E=""; else E="$e"; fi
  env $E timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-dtypes --no-c1 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$e', d['encode']['ms'], d['loopback_p2p']['ms'], d['loopback_p2p']['value'])"
done

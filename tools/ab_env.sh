#!/bin/bash
# A/B of environment settings in one GPU session: tools/ab_env.sh steps "ENV=1" "ENV=2" ...
steps=${1:-10}; shift
for rep in 1 2; do
  for e in "$@"; do
    env $e timeout 600 python bench.py --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.log 2>&1
    echo "$e rep$rep $(grep -o '"render_ms_per_step": [0-9.]*' /tmp/ab.log) $(grep -o '"value": [0-9.]*' /tmp/ab.log | head -1)"
  done
done

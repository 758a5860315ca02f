#!/bin/bash
# A/B timing of library variants in one GPU session: tools/ab.sh [steps] lib1.so lib2.so ...
steps=${1:-10}; shift
for rep in 1 2; do
  for lib in "$@"; do
    LUMI_CUDA_LIB=$lib timeout 300 python bench.py --steps $steps --warmup 3 --no-cpu-baseline --e2e-steps 1 > /tmp/ab.log 2>&1
    echo "$(basename $lib) rep$rep $(grep -o '"march_ms_per_launch": [0-9.]*' /tmp/ab.log) $(grep -o '"render_ms_per_step": [0-9.]*' /tmp/ab.log) $(grep -o '"value": [0-9.]*' /tmp/ab.log | head -1)"
  done
done

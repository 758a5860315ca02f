#!/bin/bash
# One GPU call: the -m gpu suite, the N=1 bench, the N=2 bench on the shared GPU (plumbing).
# usage (from the repo root, under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-r02}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
LUMI_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${tag}_bench_n2_shared.json 2> gpurun_out/${tag}_bench_n2_shared.err
echo "bench n2 rc=$?" >> gpurun_out/${tag}_bench_n2_shared.err
tail -5 gpurun_out/${tag}_pytest_gpu.log

#!/bin/bash
# One GPU call for kernel A/B work: parity subset on the default build, phase timing of a variant,
# then tools/ab.sh over the listed variant libraries.
#   bash tools/ab_round.sh <tag> <phase-lib or -> <lib1.so> <lib2.so> ...
tag=$1; phase=$2; shift 2
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
d=gpurun_out/ab_$tag; mkdir -p $d
if [ -n "$PARITY_LIB" ]; then
  LUMI_CUDA_LIB=$PARITY_LIB timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frame_driver.py -q -x -p no:cacheprovider --timeout 240 \
    -k "${PARITY_K:-c1 or c3_full or counts or options or c5 or odd or empty or split or gather}" > $d/pytest.log 2>&1
  echo "rc=$?" >> $d/pytest.log; tail -3 $d/pytest.log
fi
if [ "$phase" != "-" ]; then
  LUMI_CUDA_LIB=$phase timeout 200 python tools/profile_frame.py C3 1 > $d/phase.log 2>&1; grep "ws producers" $d/phase.log | head -2
fi
bash tools/ab.sh ${AB_STEPS:-10} "$@" | tee $d/ab.txt

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rP -p no:cacheprovider -k "c1 or c3_full or counts or options or gather or c5 or row_stats or golden" > gpurun_out/r02i_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02i_pytest.log
bash tools/ab.sh 10 paper_2311_02542_b200/lib/ab/nolerp.so paper_2311_02542_b200/lib/ab/lerp.so > gpurun_out/r02i_ab.txt 2>&1

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frame_driver.py -q -rP -p no:cacheprovider -k "c1 or c3_full or counts or options or c5 or odd or empty or split or concurrent or driver or zero_copy" > gpurun_out/r02k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02k_pytest.log
bash tools/ab.sh 10 paper_2311_02542_b200/lib/ab/pairs0.so paper_2311_02542_b200/lib/ab/pairs1.so > gpurun_out/r02k_ab.txt 2>&1

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frame_driver.py -q -rP -p no:cacheprovider -k "c1 or c3_full or counts or options or odd or split or empty or c5 or driver or exact_march or concurrent" > gpurun_out/r02g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02g_pytest.log
LUMI_DEBUG=1 bash tools/ab.sh 10 paper_2311_02542_b200/lib/ab/st2.so paper_2311_02542_b200/lib/ab/st3.so > gpurun_out/r02g_ab.txt 2>&1

cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frame_driver.py tests/test_gpu_train.py -q -rP -p no:cacheprovider -k "c1 or c3_full or counts or options or odd or split or empty or c5 or driver or refresh or golden" > gpurun_out/r02h_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_pytest.log
bash tools/ab_env.sh 10 "LUMI_WS_TMA=0" "LUMI_WS_TMA=1" > gpurun_out/r02h_ab.txt 2>&1

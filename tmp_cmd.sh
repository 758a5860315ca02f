cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rP -p no:cacheprovider -k "c1 or c3_full or counts or options or c5" > gpurun_out/r02j_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02j_pytest.log
bash tools/ab.sh 10 paper_2311_02542_b200/lib/ab/head.so paper_2311_02542_b200/lib/ab/split.so > gpurun_out/r02j_ab.txt 2>&1

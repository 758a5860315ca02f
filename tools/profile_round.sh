# One GPU call that refreshes the round's evidence under gpurun_out/prof/: GPU test suite, smoke,
# the bench line (C3, N=1) and the reference arm, the ncu launch list and one --set full capture of
# k_render_ws, the C5 stress line and the N=2 shared-GPU line.  Copy what is judged into profiles/.
set -x
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/prof/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/prof/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/prof/bench.json 2> gpurun_out/prof/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/prof/bench_ref.json 2> gpurun_out/prof/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_ws -c 1 -o gpurun_out/prof/ws python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof/ncu_full.log 2>&1
ls -la gpurun_out/prof
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/prof/c5.json 2>/dev/null
LUMI_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/prof/n2.json 2>/dev/null

# One GPU call that refreshes the round's evidence under gpurun_out/prof/: GPU test suite, smoke,
# the bench line (C3, N=1) and the reference arm, the ncu launch list and one --set full capture of
# k_render_ws, the march pass and the isolated MLP, the isolated gather / MLP benches, the C5
# stress line and the N=2 shared-GPU line.  Copy what is judged into profiles/.
#   bash tools/profile_round.sh <tag>
tag=${1:-r02}
set -x
cd "${GRAFT_REPO_ROOT:-.}"
d=gpurun_out/prof_$tag
mkdir -p $d
timeout 1800 python -m pytest tests -m gpu -q -rA -p no:cacheprovider > $d/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $d/smoke.log 2>&1
timeout 600 python tools/bench_gather.py > $d/bench_gather.json 2> $d/bench_gather.err
timeout 600 python tools/bench_mlp.py > $d/bench_mlp.json 2> $d/bench_mlp.err
timeout 600 python bench.py > $d/bench.json 2> $d/bench.err
timeout 900 python bench.py --impl reference > $d/bench_ref.json 2> $d/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $d/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $d/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render_ws -c 1 -o $d/ws python tools/profile_frame.py C3 1 > $d/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_march_seg -c 1 -o $d/march python tools/profile_frame.py C3 1 > $d/ncu_march.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_mlp_batch -c 1 -o $d/mlp python tools/bench_mlp.py --steps 1 > $d/ncu_mlp.log 2>&1
timeout 900 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $d/c5.json 2> $d/c5.err
LUMI_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $d/n2.json 2> $d/n2.err
ls -la $d

# usage: bash scripts/gpu_prof.sh TAG -- build, gpu tests, bench, ncu launch list + full capture
cd $GRAFT_REPO_ROOT
TAG=${1:-r}
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?; cat gpurun_out/bench_$TAG.json | cut -c1-3000
./scripts/microbench > gpurun_out/microbench.txt 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench scripts/microbench.cu && ./scripts/microbench > gpurun_out/microbench.txt)
timeout -s KILL 300 python scripts/k1_timeline.py --out gpurun_out/k1_timeline_$TAG.json > /dev/null 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 --csv \
    --log-file gpurun_out/launches_$TAG.csv python scripts/profile_epoch.py --epochs 8 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu-launch rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k1_sweep|k4_assign" -s 2 -c 2 \
    -o gpurun_out/prof_$TAG python scripts/profile_epoch.py --epochs 3 > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu-full rc=$?

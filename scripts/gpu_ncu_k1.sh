# usage: bash scripts/gpu_ncu_k1.sh TAG -- one ncu --set full capture of K1 + K4 (source-level), C4 table
cd $GRAFT_REPO_ROOT
TAG=${1:-k}
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout -s KILL 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"k1_sweep|k4_assign" -s 2 -c 2 \
    -o gpurun_out/prof_$TAG python scripts/profile_epoch.py --epochs 3 > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu-full rc=$?

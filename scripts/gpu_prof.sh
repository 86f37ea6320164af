# usage: bash scripts/gpu_prof.sh TAG   -- tests, bench, ncu launch list + full capture of K1 and K4
cd $GRAFT_REPO_ROOT
TAG=${1:-r}
bash scripts/gpu_check.sh
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 10 -c 20 --csv \
    --log-file gpurun_out/launches_$TAG.csv python scripts/profile_epoch.py --epochs 8 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo ncu-launch rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k1_sweep|k4_assign" -s 2 -c 2 \
    -o gpurun_out/prof_$TAG python scripts/profile_epoch.py --epochs 3 > gpurun_out/ncu_full_$TAG.log 2>&1; echo ncu-full rc=$?
tail -3 gpurun_out/ncu_full_$TAG.log

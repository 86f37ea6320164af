# usage: bash scripts/gpu_base.sh TAG -- gpu_prof.sh plus ncu launch list + dram bytes at C5 (2^20)
cd $GRAFT_REPO_ROOT
TAG=${1:-r}
bash scripts/gpu_prof.sh $TAG
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 12 -c 12 --csv \
    --log-file gpurun_out/launches_c5_$TAG.csv python scripts/profile_epoch.py --n 1048576 --epochs 8 > gpurun_out/ncu_launch_c5_$TAG.log 2>&1; echo ncu-c5 rc=$?

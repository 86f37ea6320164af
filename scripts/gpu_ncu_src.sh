# usage: bash scripts/gpu_ncu_src.sh KERNEL_REGEX TAG -- ncu --set full (dense warp sampling,
# source-level) of one launch of the kernel in a C4 epoch; raw + source csv into gpurun_out/
cd $GRAFT_REPO_ROOT
K=$1; TAG=$2
timeout -s KILL 300 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"$K" -s 2 -c 1 \
    -o gpurun_out/src_$TAG python scripts/profile_epoch.py --epochs 3 > gpurun_out/src_$TAG.log 2>&1; echo rc=$?
ncu -i gpurun_out/src_$TAG.ncu-rep --page raw --csv > gpurun_out/src_${TAG}_raw.csv 2>&1
ncu -i gpurun_out/src_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_src.csv 2>&1

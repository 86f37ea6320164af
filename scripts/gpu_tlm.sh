cd $GRAFT_REPO_ROOT
./scripts/microbench || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench scripts/microbench.cu && ./scripts/microbench)
bash scripts/gpu_tl.sh

cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/codeptr scripts/codeptr_probe.cu && timeout 60 /tmp/codeptr > gpurun_out/codeptr.txt 2>&1
timeout -s KILL 600 python scripts/code_warm_ab.py > gpurun_out/code_warm.txt 2>&1
cat gpurun_out/codeptr.txt gpurun_out/code_warm.txt

cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/latency_probe scripts/latency_probe.cu && timeout 120 /tmp/latency_probe > gpurun_out/latency_probe.txt 2>&1
timeout -s KILL 600 python scripts/epoch_anatomy.py > gpurun_out/anatomy.log 2>&1
timeout -s KILL 600 python bench.py --steps 300 --warmup 10 --cpu-budget 1 --e2e-steps 50 > gpurun_out/bench0.json 2> gpurun_out/bench0.err
echo done

cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
NCCL_DEBUG=WARN timeout -s KILL 300 python -m pytest tests/test_parity_gpu.py -m gpu -q -k nccl -p no:cacheprovider 2>&1 | tail -30
timeout -s KILL 600 python bench.py --steps 50 --warmup 10 --cpu-budget 1 --e2e-steps 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d.get('c3_dynamic')); print(d['value'], d['kernels_us'])" || tail -20 gpurun_out/bench.err

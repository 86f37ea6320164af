# usage: bash scripts/gpu_tl.sh -- build, K1/K4 timeline, short bench (no tests)
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout -s KILL 300 python scripts/k1_timeline.py > gpurun_out/timeline.log 2>&1; python -c "
import json; d=json.load(open('gpurun_out/k1_timeline.json')); print({k:v for k,v in d.items() if k!='slowest'}); print(d['slowest'][:2])" || tail gpurun_out/timeline.log
timeout -s KILL 600 python bench.py --steps 50 --warmup 10 --cpu-budget 1 --e2e-steps 5 2> gpurun_out/bench.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('value','ms_per_step','kernels_us','epoch_us_p50','e2e')})"

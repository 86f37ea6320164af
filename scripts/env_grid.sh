# usage: bash scripts/env_grid.sh "ENV=a" "ENV=b" ... -- C4 epoch under several environments, interleaved, 2 rounds
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --steps 600 --c3-epochs 0 --cpu-budget 0 --e2e-steps 5 > gpurun_out/eg.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/eg.json'));print('$e', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2), 'k1', round(d['kernels_us']['k1_sweep'],2), 'k4', round(d['kernels_us']['k4_assign'],2))"
  done
done

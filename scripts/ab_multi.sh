# usage: bash scripts/ab_multi.sh A.so B.so ... -- C4 epoch of several in-tree builds, interleaved, 3 rounds
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  for lib in "" "$@"; do
    env NALAR_LIB_AB=$lib timeout 300 python bench.py --steps 800 --c3-epochs 0 --cpu-budget 0 > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('${lib:-head}', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2), 'k1', round(d['kernels_us']['k1_sweep'],2), 'k4', round(d['kernels_us']['k4_assign'],2), 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"
  done
done

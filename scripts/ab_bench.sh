# usage: bash scripts/ab_bench.sh libA.so libB.so -- the C4 bench line (mean / p50 / p99 epoch) of two
# in-tree builds, alternating, 3 reps each
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  for lib in "$@"; do
    NALAR_LIB_AB=$lib timeout 300 python bench.py --steps 2000 --c3-epochs 0 --cpu-budget 0 --c5 0 --c4-survey 0 --e2e-steps 5 > gpurun_out/abb.json 2>/dev/null
    [ -s gpurun_out/abb.json ] && python -c "import json;d=json.load(open('gpurun_out/abb.json'));print('$lib', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2), 'p99', round(d['epoch_us_p99'],2))"
  done
done

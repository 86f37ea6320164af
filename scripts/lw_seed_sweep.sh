# usage: bash scripts/lw_seed_sweep.sh "w1 w2 ..." "seed1 seed2" -- epoch per long-workflow partition weight and table seed
cd $GRAFT_REPO_ROOT
for seed in $2; do
  for v in $1; do
    NALAR_LONG_WEIGHT=$v timeout 300 python bench.py --steps 600 --c3-epochs 0 --cpu-budget 0 --seed $seed > gpurun_out/es.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/es.json'));print('seed $seed weight $v', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2))"
  done
done

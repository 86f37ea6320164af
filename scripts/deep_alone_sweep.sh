# usage: bash scripts/deep_alone_sweep.sh -- epoch vs giving deep workflows a block of their own, over table seeds
cd $GRAFT_REPO_ROOT
for seed in ${SEEDS:-1 2 3}; do
  for v in ${VALS:-0 12 16 20}; do
    NALAR_DEEP_ALONE=$v timeout 300 python bench.py --steps 600 --c3-epochs 0 --cpu-budget 0 --seed $seed > gpurun_out/es.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/es.json'));print('seed $seed deep_alone $v', round(d['ms_per_step']*1e3,2))"
  done
done

cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for cfg in "NALAR_K1_BLOCKS=142" "NALAR_K1_BLOCKS=144" "NALAR_K1_BLOCKS=146" "NALAR_K1_BLOCKS=140"; do
  env $cfg timeout 300 python bench.py --steps 800 --c3-epochs 0 --cpu-budget 0 > gpurun_out/es.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/es.json'));print('$cfg', round(d['ms_per_step']*1e3,2))"
done
done

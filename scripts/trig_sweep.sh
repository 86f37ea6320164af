cd $GRAFT_REPO_ROOT
for cfg in "NALAR_K4_PDL=0 NALAR_K1_TRIGGER=0" "NALAR_K4_PDL=1 NALAR_K1_TRIGGER=0" "NALAR_K4_PDL=1 NALAR_K1_TRIGGER=1" "NALAR_K4_PDL=1 NALAR_K1_TRIGGER=2"; do
  for rep in 1 2; do
    env $cfg timeout 300 python bench.py --steps 800 --c3-epochs 0 --cpu-budget 0 > gpurun_out/es.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/es.json'));print('$cfg', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2))"
  done
done

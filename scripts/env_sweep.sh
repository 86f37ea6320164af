# usage: bash scripts/env_sweep.sh VAR "v1 v2 ..." -- bench epoch per env setting (2 repeats each)
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > /dev/null 2>&1
VAR=$1
for v in $2; do
  for rep in 1 2; do
    env $VAR=$v timeout 300 python bench.py --steps 800 --c3-epochs 0 --cpu-budget 0 > gpurun_out/es.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/es.json'));print('$VAR=$v', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2), 'k1', round(d['kernels_us']['k1_sweep'],2), 'k4', round(d['kernels_us']['k4_assign'],2))"
  done
done

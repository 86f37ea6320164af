# partition knobs A/B: NALAR_FILL_SMS (grow blocks to fill the SMs) x NALAR_LONG_WEIGHT
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > /dev/null 2>&1
for cfg in "0 1.0" "1 1.0" "1 0.7" "1 1.3"; do
  set -- $cfg
  NALAR_FILL_SMS=$1 NALAR_LONG_WEIGHT=$2 timeout 300 python bench.py --steps 600 --c3-epochs 0 --cpu-budget 0 > gpurun_out/lw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/lw.json'));print('fill $1 lw $2', round(d['ms_per_step']*1e3,2), 'k1', round(d['kernels_us']['k1_sweep'],2), 'e2e', round(d['e2e']['ms_per_step']*1e3,1))"
done

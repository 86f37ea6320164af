# quick A/B bench (3 repeats)
cd $GRAFT_REPO_ROOT
python paper_2601_05109_b200/build.py > /dev/null 2>&1
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 800 --c3-epochs 0 --cpu-budget 0 > gpurun_out/lw.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/lw.json'));print('run', round(d['ms_per_step']*1e3,2), 'k1', round(d['kernels_us']['k1_sweep'],2), 'k4', round(d['kernels_us']['k4_assign'],2))"
done

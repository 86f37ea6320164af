# usage: bash scripts/e2e_ab.sh -- e2e A/B: the in-tree libnalar.so vs libnalar_base.so (build it from another commit)
cd $GRAFT_REPO_ROOT
timeout -s KILL 600 python -m pytest tests/test_io_gpu.py tests/test_step_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2 3; do for lib in "" libnalar_base.so; do
  env NALAR_LIB_AB=$lib timeout 300 python bench.py --steps 300 --c3-epochs 0 --cpu-budget 0 --e2e-steps 60 > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('${lib:-new}', round(d['e2e']['ms_per_step']*1e3,1), round(d['e2e']['split_calls_ms_per_step']*1e3,1), d['e2e']['parts'])"
done; done

# usage: bash scripts/ab.sh [B.so] -- A/B bench: the in-tree libnalar.so vs another in-tree build
# (default libnalar_base.so), alternating, 3 runs each, plus one K1 timeline of each
cd $GRAFT_REPO_ROOT
B=${1:-libnalar_base.so}
for rep in 1 2 3; do
  for lib in "" $B; do
    env NALAR_LIB_AB=$lib timeout 300 python bench.py --steps 800 --c3-epochs 0 --cpu-budget 0 > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('${lib:-new}', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2), 'k1', round(d['kernels_us']['k1_sweep'],2), 'k4', round(d['kernels_us']['k4_assign'],2))"
  done
done
for lib in "" $B; do
  env NALAR_LIB_AB=$lib timeout 300 python scripts/k1_timeline.py --out gpurun_out/ab_tl_${lib:-new}.json > /dev/null 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/ab_tl_${lib:-new}.json'))
print('${lib:-new}', {k:d[k] for k in ('kernel_span_ns','sweep_ns_max','wf_end_ns_max','p3_ns_max','p5_ns_max','bucket_ns_max','p2_end_ns_pct')}, d['transfer_steps']['cycles_per_step'])"
done

# usage: bash scripts/ab_env.sh "ENV=a" "ENV=b" -- A/B bench of one build under two environments, 3 runs each + timelines
cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  for e in "$1" "$2"; do
    env $e timeout 300 python bench.py --steps 800 --c3-epochs 0 --cpu-budget 0 > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$e', round(d['ms_per_step']*1e3,2), 'p50', round(d['epoch_us_p50'],2), 'k1', round(d['kernels_us']['k1_sweep'],2), 'k4', round(d['kernels_us']['k4_assign'],2))"
  done
done
for e in "$1" "$2"; do
  tag=$(echo "$e" | tr '= ' '__')
  env $e timeout 300 python scripts/k1_timeline.py --out gpurun_out/abe_tl_$tag.json > /dev/null 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/abe_tl_$tag.json'))
print('$e', {k:d[k] for k in ('kernel_span_ns','sweep_ns_max','wf_end_ns_max','p3_ns_max','p5_ns_max','bucket_ns_max','p2_end_ns_pct')})
for w in d['slowest'][:4]: print('   ', w)"
done

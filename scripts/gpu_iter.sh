# usage: bash scripts/gpu_iter.sh TAG -- quick iteration: build, GPU parity tests, short bench, K1 timelines
cd $GRAFT_REPO_ROOT
TAG=${1:-it}
python paper_2601_05109_b200/build.py > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
timeout -s KILL 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 300 python bench.py --steps 1000 --c3-epochs 0 --cpu-budget 0 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print('epoch_us',d['ms_per_step']*1e3,'p50',d['epoch_us_p50'],'kernels',d['kernels_us'],'e2e_ms',d['e2e']['ms_per_step'])"
timeout -s KILL 300 python scripts/k1_timeline.py --out gpurun_out/k1_timeline_$TAG.json > /dev/null 2>&1
timeout -s KILL 300 python scripts/k1_cta_detail.py --out gpurun_out/k1_cta_$TAG.json > /dev/null 2>&1
python -c "
import json;d=json.load(open('gpurun_out/k1_timeline_$TAG.json'));print({k:v for k,v in d.items() if k not in ('slowest','blocks')})
c=json.load(open('gpurun_out/k1_cta_$TAG.json'))
for x in c['ctas'][:3]: print({k:v for k,v in x.items() if k!='wfs'}); [print('   ',w) for w in x['wfs']]
"

# usage: bash scripts/gpu_quick.sh <tag> [extra bench args] : build, GPU tests, bench lines at 128K, 1M and 32K bs8
cd $GRAFT_REPO_ROOT
tag=${1:-q}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 300 > gpurun_out/pytest_$tag.log 2>&1
tail -3 gpurun_out/pytest_$tag.log
for c in 128k 1m 32k_bs8; do
  st=200; [ $c = 1m ] && st=20; [ $c = 32k_bs8 ] && st=100
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu --no-dense "$@" > gpurun_out/bench_${tag}_$c.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/bench_${tag}_$c.log').read().strip().splitlines()[-1]);print('$c', d['value'], d['e2e']['value'], {k:v['avg_us'] for k,v in d['kernels'].items()})" || tail -5 gpurun_out/bench_${tag}_$c.log
done
echo done

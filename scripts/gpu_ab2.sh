# usage: bash scripts/gpu_ab2.sh "<ENV=val ...>" ... : bench A/B (3 runs each, interleaved)
cd $GRAFT_REPO_ROOT
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
for r in 1 2; do
for envs in "$@"; do
  env $envs timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-dense > /tmp/ab.log 2>&1
  echo "[$envs] $(python -c "import json,sys;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);print(d['value'], {k:v['avg_us'] for k,v in d['kernels'].items()})")"
done; done

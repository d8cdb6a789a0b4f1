# usage: bash scripts/gpu_ab3.sh <config> "<ENV=val ...>" ... : bench A/B on one config (2 rounds, interleaved)
cd $GRAFT_REPO_ROOT
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
cfg=$1; shift
for r in 1 2; do
for envs in "$@"; do
  env $envs timeout 600 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu --no-dense > /tmp/ab.log 2>&1
  echo "[$cfg $envs] $(python -c "import json,sys;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);print(d['value'], {k:v['avg_us'] for k,v in d['kernels'].items()})")"
done; done

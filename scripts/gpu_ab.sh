# usage: bash scripts/gpu_ab.sh <tag> "<ENV=val ...>" ["<ENV=val ...>" ...] : bench A/B over environment settings
cd $GRAFT_REPO_ROOT
tag=$1; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
i=0
for envs in "$@"; do
  env $envs timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-dense > gpurun_out/ab_${tag}_$i.log 2>&1
  echo "[$envs] $(python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${tag}_$i.log').read().strip().splitlines()[-1]);print(d['value'], {k:v['avg_us'] for k,v in d['kernels'].items()})")"
  i=$((i+1))
done

# usage: bash scripts/gpu_envab.sh <tag> <config> <steps> "<ENV=val ...>" ... : bench env-switch variants one after another
cd $GRAFT_REPO_ROOT
tag=$1; cfg=$2; st=$3; shift 3
mkdir -p gpurun_out
i=0
for envs in "$@"; do
  env $envs timeout 600 python bench.py --config $cfg --steps $st --warmup 5 --no-cpu --no-dense --no-1m > gpurun_out/ab_${tag}_$i.log 2>&1
  echo "[$envs] $(python -c "
import json;d=json.loads(open('gpurun_out/ab_${tag}_$i.log').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], {k: v['avg_us'] for k, v in d['kernels'].items()})" 2>&1 | tail -1)"
  i=$((i+1))
done

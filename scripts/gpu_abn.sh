# usage: bash scripts/gpu_abn.sh <tag> <config> <reps> "<ENV=val ...>" ... : alternating bench A/B (reps rounds)
cd $GRAFT_REPO_ROOT
tag=$1; cfg=$2; reps=$3; shift 3
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
st=200; [ $cfg = 1m ] && st=30
for r in $(seq 1 $reps); do
  i=0
  for envs in "$@"; do
    env $envs timeout 600 python bench.py --config $cfg --steps $st --warmup 5 --no-cpu --no-dense > gpurun_out/abn_${tag}_${r}_$i.log 2>&1
    echo "r$r [$envs] $(python -c "import json,sys;d=json.loads(open('gpurun_out/abn_${tag}_${r}_$i.log').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'])")"
    i=$((i+1))
  done
done

cd $GRAFT_REPO_ROOT
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
for envs in "$@"; do
  env $envs timeout 900 python bench.py --config 1m --steps 20 --warmup 3 --no-cpu > /tmp/w.log 2>&1; echo "[1m $envs] $(python -c "import json;d=json.loads(open('/tmp/w.log').read().strip().splitlines()[-1]);print(d['value'], {k:v['avg_us'] for k,v in d['kernels'].items()})")"
done

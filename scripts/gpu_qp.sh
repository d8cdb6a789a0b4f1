cd $GRAFT_REPO_ROOT
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for r in 1 2; do
for c in 128k 32k_bs8; do
  timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu --no-dense > /tmp/ab.log 2>&1
  echo "[$c] $(python -c "import json,sys;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], {k:v['avg_us'] for k,v in d['kernels'].items()})")"
done; done

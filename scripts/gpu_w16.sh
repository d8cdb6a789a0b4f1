cd $GRAFT_REPO_ROOT
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 600 2>&1 | tail -3
for a in "" "--w16" "" "--w16"; do timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-dense $a > /tmp/w.log 2>&1; echo "[$a] $(python -c "import json;d=json.loads(open('/tmp/w.log').read().strip().splitlines()[-1]);print(d['value'], {k:v['avg_us'] for k,v in d['kernels'].items()})")"; done
for a in "" "--w16"; do timeout 900 python bench.py --config 1m --steps 20 --warmup 3 --no-cpu $a > /tmp/w.log 2>&1; echo "[1m $a] $(python -c "import json;d=json.loads(open('/tmp/w.log').read().strip().splitlines()[-1]);print(d['value'], {k:v['avg_us'] for k,v in d['kernels'].items()})")"; done

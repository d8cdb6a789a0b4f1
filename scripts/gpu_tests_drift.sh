cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_td.log 2>&1 || { tail -30 gpurun_out/build_td.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 600 > gpurun_out/pytest_td.log 2>&1
tail -15 gpurun_out/pytest_td.log
timeout 900 python scripts/drift_recall.py --prefill 8192 --decode 4096 --rates 0,0.002,0.01 --out gpurun_out/drift_small.json 2>&1 | tail -5

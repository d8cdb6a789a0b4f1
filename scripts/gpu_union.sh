# usage: bash scripts/gpu_union.sh : GQA-union rerank parity test + A/B against the per-head kernel
cd $GRAFT_REPO_ROOT
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_ab3.sh 128k X=0 PKV_RERANK=union "PKV_RERANK=union PKV_LIB=u8"
bash scripts/gpu_ab3.sh 1m X=0 PKV_RERANK=union

# usage: bash scripts/gpu_tests.sh <tag> [pytest -k expr] : build + the -m gpu suite + smoke
cd $GRAFT_REPO_ROOT
tag=${1:-t}; kexpr=${2:-}
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
if [ -n "$kexpr" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 1200 -k "$kexpr" > gpurun_out/pytest_$tag.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/pytest_$tag.log 2>&1
fi
tail -30 gpurun_out/pytest_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; tail -3 gpurun_out/smoke_$tag.log

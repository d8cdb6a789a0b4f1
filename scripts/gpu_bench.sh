# usage: bash scripts/gpu_bench.sh <tag> [extra bench args] : the default bench line (128K + 1M block + CPU oracle)
cd $GRAFT_REPO_ROOT
tag=${1:-b}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
start=$(date +%s)
timeout 1500 python bench.py "$@" > gpurun_out/bench_$tag.log 2> gpurun_out/bench_${tag}_err.log
echo "rc=$? wall_s=$(( $(date +%s) - start ))"
tail -c 3000 gpurun_out/bench_$tag.log; echo
tail -5 gpurun_out/bench_${tag}_err.log

# usage: bash scripts/gpu_sanitize.sh <tag> : compute-sanitizer memcheck / racecheck / synccheck over smoke() and
#   selected GPU tests; logs under gpurun_out/san_<tag>_*.txt (copy the final set to profiles/)
cd $GRAFT_REPO_ROOT
tag=${1:-s}
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
CS="compute-sanitizer --print-limit 20"
run() {  # name tool pytest-k
  timeout 1500 $CS --tool $2 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$3" > gpurun_out/san_${tag}_$1.txt 2>&1
  echo "$1 ($2, -k '$3'): $(grep -E 'passed|failed' gpurun_out/san_${tag}_$1.txt | tail -1) | $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|SYNCCHECK SUMMARY' gpurun_out/san_${tag}_$1.txt | tail -1)"
}
timeout 600 $CS --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${tag}_smoke_memcheck.txt 2>&1
echo "smoke memcheck: $(grep -E 'smoke OK|ERROR SUMMARY' gpurun_out/san_${tag}_smoke_memcheck.txt | tr '\n' ' ')"
run seg_racecheck racecheck "segmented and 150000"
run seg_memcheck memcheck "segmented"
run stream_memcheck memcheck "stream"
run keyfrac_memcheck memcheck "key_fraction"
run gqa_racecheck racecheck "gqa_batch_ragged or massive_estimate_ties or fused_exchange"
run gqa_synccheck synccheck "gqa_batch_ragged or massive_estimate_ties"

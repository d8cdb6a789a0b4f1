# usage: bash scripts/gpu_evidence.sh <tag> : the committed evidence set of one build — GPU suite + smoke, the default
#   bench line (128K + 1M block + CPU oracle), 32K bs8, key-fraction and 1M keys-in-HBM lines, the phase anatomy at
#   128K and 1M, warm ncu launch lists and one `ncu --set full` capture of a layer at 128K and 1M
cd $GRAFT_REPO_ROOT
tag=${1:-ev}
mkdir -p gpurun_out
bash scripts/gpu_tests.sh $tag
run() {  # name args...
  local name=$1; shift
  timeout 1200 python bench.py "$@" > gpurun_out/bench_${tag}_$name.log 2> gpurun_out/bench_${tag}_${name}_err.log
  echo "$name rc=$? $(tail -c 300 gpurun_out/bench_${tag}_$name.log | tr -d '\n' | cut -c1-200)"
}
run 128k_with_1m
run 32k_bs8 --config 32k_bs8 --no-cpu
run 128k_key_fraction --key-fraction --no-cpu --no-1m
run 1m_khbm --config 1m --k-hbm --no-cpu
bash scripts/gpu_phase.sh $tag > /dev/null 2>&1
unset PKV_PHASE_PROFILE PKV_LIB_TAG PKV_LIB
bash scripts/gpu_prof.sh $tag warm > /dev/null 2>&1
bash scripts/gpu_prof.sh $tag full > /dev/null 2>&1
ls gpurun_out | grep "_$tag" | head -40

# usage: bash scripts/gpu_phase.sh <tag> : phase anatomy only (profiling build), then restore the product build
cd $GRAFT_REPO_ROOT
tag=${1:-ph}
mkdir -p gpurun_out
PKV_PHASE_PROFILE=1 timeout 300 python scripts/phase_profile.py > gpurun_out/phase_$tag.txt 2>&1
tail -12 gpurun_out/phase_$tag.txt

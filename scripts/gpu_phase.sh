# usage: bash scripts/gpu_phase.sh <tag> [ENV=val ...] : kernel anatomy (globaltimer marks, profiling build
#   libpariskv_phase.so, one layer replayed from a CUDA graph) at 128K and 1M
cd $GRAFT_REPO_ROOT
tag=${1:-ph}; shift
mkdir -p gpurun_out
export PKV_PHASE_PROFILE=1 PKV_LIB_TAG=phase PKV_LIB=phase
env "$@" timeout 300 python scripts/phase_profile.py > gpurun_out/phase_${tag}_128k.txt 2>&1
PHASE_CTX=1048576 PHASE_UVA=1 env "$@" timeout 600 python scripts/phase_profile.py > gpurun_out/phase_${tag}_1m.txt 2>&1
head -6 gpurun_out/phase_${tag}_128k.txt; head -6 gpurun_out/phase_${tag}_1m.txt

# usage: bash scripts/gpu_phase.sh <tag> : kernel anatomy (globaltimer marks, profiling build libpariskv_phase.so) at 128K and 1M
cd $GRAFT_REPO_ROOT
tag=${1:-ph}
mkdir -p gpurun_out
export PKV_PHASE_PROFILE=1 PKV_LIB_TAG=phase PKV_LIB=phase
timeout 300 python scripts/phase_profile.py > gpurun_out/phase_${tag}_128k.txt 2>&1
PHASE_CTX=1048576 PHASE_UVA=1 timeout 600 python scripts/phase_profile.py > gpurun_out/phase_${tag}_1m.txt 2>&1
tail -12 gpurun_out/phase_${tag}_128k.txt

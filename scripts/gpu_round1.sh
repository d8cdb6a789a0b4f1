set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
python -m paper_2602_07721_b200.build > gpurun_out/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 400 > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 50 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log

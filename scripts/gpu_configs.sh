# usage: bash scripts/gpu_configs.sh <tag> : bench lines for the 32k_bs8 and 1M configs
cd $GRAFT_REPO_ROOT
tag=${1:-cfg}
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 900 python bench.py --config 32k_bs8 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_${tag}_32k.log 2>&1
tail -c 300 gpurun_out/bench_${tag}_32k.log
timeout 1200 python bench.py --config 1m --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_${tag}_1m.log 2>&1
tail -c 300 gpurun_out/bench_${tag}_1m.log

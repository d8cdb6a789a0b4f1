# usage: bash scripts/gpu_iter2.sh <tag> : tests, bench, phase anatomy, warm ncu launch list
cd $GRAFT_REPO_ROOT
tag=${1:-it}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 300 > gpurun_out/pytest_$tag.log 2>&1
tail -3 gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu "$@" > gpurun_out/bench_$tag.log 2>&1
tail -c 300 gpurun_out/bench_$tag.log
PKV_PHASE_PROFILE=1 timeout 300 python scripts/phase_profile.py > gpurun_out/phase_$tag.txt 2>&1
tail -9 gpurun_out/phase_$tag.txt
python -m paper_2602_07721_b200.build > /dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_${tag}_warm.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu --no-dense > /dev/null 2>&1
echo done

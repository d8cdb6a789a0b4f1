# usage: bash scripts/gpu_prof.sh <tag> : parity tests, bench, ncu launch list, ncu --set full of each hot kernel
cd $GRAFT_REPO_ROOT
tag=${1:-p}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_$tag.log 2>&1
tail -3 gpurun_out/pytest_$tag.log
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu "$@" > gpurun_out/bench_$tag.log 2>&1
tail -c 600 gpurun_out/bench_$tag.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_kernel|topk_kernel|attend_partial" -s 12 -c 6 -o gpurun_out/prof_$tag python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_full_$tag.log 2>&1
echo done

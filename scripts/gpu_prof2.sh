cd $GRAFT_REPO_ROOT
tag=${1:-p}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_kernel|topk_kernel|attend_partial" -s 18 -c 6 -o gpurun_out/prof_$tag python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_full_$tag.log 2>&1
echo done

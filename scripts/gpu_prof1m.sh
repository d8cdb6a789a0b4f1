# usage: bash scripts/gpu_prof1m.sh <tag> : ncu --set full of the per-step kernels at the 1M configuration
cd $GRAFT_REPO_ROOT
tag=${1:-p1m}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_cpt_kernel|topk_cl_kernel" -s 10 -c 5 -o gpurun_out/prof_$tag python bench.py --config 1m --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense "$@" > gpurun_out/ncu_full_$tag.log 2>&1
python scripts/ncu_full_summary.py gpurun_out/prof_$tag.ncu-rep "ncu --set full, 1M config ($tag)" > gpurun_out/ncu_full_${tag}_summary.txt 2>&1
cat gpurun_out/ncu_full_${tag}_summary.txt | tail -8
echo done

# usage: bash scripts/gpu_prof_q.sh <tag> : ncu --set full of the per-step kernels at 1M and 128K + host-link microbench
cd $GRAFT_REPO_ROOT
tag=${1:-pq}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/uva_bw scripts/uva_bw.cu && timeout 300 /tmp/uva_bw > gpurun_out/uva_bw_$tag.txt 2>&1; cat gpurun_out/uva_bw_$tag.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"scan_kernel|select_kernel|rerank_cpt_kernel|topk_cl_kernel" -s 8 -c 4 -o gpurun_out/prof_${tag}_1m python bench.py --config 1m --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense "$@" > gpurun_out/ncu_full_${tag}_1m.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_cpt_kernel|topk_cl_kernel" -s 10 -c 5 -o gpurun_out/prof_${tag}_128k python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense "$@" > gpurun_out/ncu_full_${tag}_128k.log 2>&1
for c in 1m 128k; do python scripts/ncu_full_summary.py gpurun_out/prof_${tag}_$c.ncu-rep "ncu --set full, $c ($tag)" > gpurun_out/ncu_full_${tag}_${c}_summary.txt 2>&1; tail -6 gpurun_out/ncu_full_${tag}_${c}_summary.txt; done
echo done

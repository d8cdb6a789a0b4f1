# usage: bash scripts/gpu_ncu_qprep.sh : ncu --set full of one qprep launch at 32k bs8
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|rerank_cpt_kernel" -s 4 -c 2 -o gpurun_out/prof_qp python bench.py --config 32k_bs8 --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense > gpurun_out/ncu_qp.log 2>&1
python scripts/ncu_full_summary.py gpurun_out/prof_qp.ncu-rep qp > gpurun_out/prof_qp.txt 2>&1
ncu -i gpurun_out/prof_qp.ncu-rep --page source --csv -k regex:qprep > gpurun_out/prof_qp_src.csv 2>/dev/null
cat gpurun_out/prof_qp.txt

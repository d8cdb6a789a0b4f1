cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 3 --no-cpu > gpurun_out/bench2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v1.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_run.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"scan_kernel|rerank_kernel|compact_kernel|topk_kernel|qprep_kernel|threshold_kernel|attend_partial|encode_kernel" -c 8 -o gpurun_out/prof_v1 python bench.py --layers 1 --steps 1 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_full_run.log 2>&1
ls -la gpurun_out

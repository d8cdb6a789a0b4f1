# usage: bash scripts/gpu_full.sh <tag> : ncu --set full capture of one layer's kernels, all bench configs,
# the contract bench line (with the CPU oracle baseline) and the reference (oracle) arm
cd $GRAFT_REPO_ROOT
tag=${1:-full}; shift
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_kernel|topk_kernel" -s 15 -c 5 -o gpurun_out/prof_$tag python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense > gpurun_out/ncu_full_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/prof_${tag}_raw.csv 2>&1
timeout 900 python bench.py --steps 200 --warmup 5 > gpurun_out/bench_${tag}_128k.log 2>&1
tail -c 400 gpurun_out/bench_${tag}_128k.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${tag}_ref.log 2>&1
tail -c 300 gpurun_out/bench_${tag}_ref.log
timeout 900 python bench.py --config 32k_bs8 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_${tag}_32k.log 2>&1
tail -c 300 gpurun_out/bench_${tag}_32k.log
timeout 1200 python bench.py --config 1m --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_${tag}_1m.log 2>&1
tail -c 300 gpurun_out/bench_${tag}_1m.log
echo done

# usage: bash scripts/gpu_ncu_src.sh <tag> "<kernel regex>" : ncu --set full with source for one launch of each kernel
cd $GRAFT_REPO_ROOT
tag=$1; rx=$2
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s 10 -c 4 -o gpurun_out/prof_$tag python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense > gpurun_out/ncu_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
echo done

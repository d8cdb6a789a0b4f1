# usage: bash scripts/gpu_prof.sh <tag> [what] : ncu evidence for DESIGN/profiles
#   what=scan1m : ncu --set full of one warm scan launch at 1M (L1 wavefront budget)
#   what=full   : ncu --set full of one layer's five kernels at 128K and 1M
#   what=warm   : warm launch lists (gpu__time_duration, no cache flush) at 128K and 1M
cd $GRAFT_REPO_ROOT
tag=${1:-p}; what=${2:-warm}
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
B="python bench.py --steps 1 --warmup 3 --no-cpu --no-dense --no-1m"
if [ "$what" = scan1m ] || [ "$what" = all ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_kernel -s 8 -c 1 -o gpurun_out/scan1m_$tag $B --config 1m --layers 4 --no-graph > gpurun_out/ncu_scan1m_$tag.log 2>&1
  ncu -i gpurun_out/scan1m_$tag.ncu-rep --page raw --csv > gpurun_out/scan1m_${tag}_raw.csv 2>/dev/null
  ncu -i gpurun_out/scan1m_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/scan1m_${tag}_sass.csv 2>/dev/null
fi
if [ "$what" = full ] || [ "$what" = all ]; then
  for c in 128k 1m; do
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_cpt_kernel|rerank_flat_kernel|topk_cl_kernel" -s 10 -c 5 -o gpurun_out/full_${c}_$tag $B --config $c --layers 4 --no-graph > gpurun_out/ncu_full_${c}_$tag.log 2>&1
    ncu -i gpurun_out/full_${c}_$tag.ncu-rep --page raw --csv > gpurun_out/full_${c}_${tag}_raw.csv 2>/dev/null
  done
fi
if [ "$what" = warm ] || [ "$what" = all ]; then
  for c in 128k 1m; do
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_${c}_${tag}.csv $B --config $c --layers 4 > /dev/null 2>&1
  done
fi
ls -la gpurun_out | tail -20

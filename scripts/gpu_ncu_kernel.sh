# usage: bash scripts/gpu_ncu_kernel.sh <tag> <config> <kernel-regex> <lib-variant>... : one `ncu --set full` capture
#   of one warm launch of the kernel per library variant ("base" = libpariskv.so), raw CSV exported for reading here
cd $GRAFT_REPO_ROOT
tag=$1; cfg=$2; kre=$3; shift 3
mkdir -p gpurun_out
for v in "$@"; do
  lib=$v; [ $v = base ] && lib=
  PKV_LIB=$lib timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$kre" -s ${SKIP:-8} -c 1 \
    -o gpurun_out/ncu_${tag}_$v python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu --no-dense --no-1m \
    --layers 4 --no-graph > gpurun_out/ncu_${tag}_$v.log 2>&1
  ncu -i gpurun_out/ncu_${tag}_$v.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_${v}_raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu_${tag}_$v.ncu-rep --page details --csv > gpurun_out/ncu_${tag}_${v}_det.csv 2>/dev/null
  ncu -i gpurun_out/ncu_${tag}_$v.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${tag}_${v}_sass.csv 2>/dev/null
  ncu -i gpurun_out/ncu_${tag}_$v.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu_${tag}_${v}_cuda.csv 2>/dev/null
  echo "$v: $(grep -c . gpurun_out/ncu_${tag}_${v}_raw.csv) raw lines"
done

# usage: bash scripts/gpu_variants.sh <tag> <config> <steps> <lib-variant>... : bench the prebuilt library variants
#   (libpariskv_<v>.so, built here with PKV_LIB_TAG=<v> PKV_BUILD_DEFS=...; "base" = libpariskv.so) one after
#   another on the same box, printing value, e2e and per-kernel event times
cd $GRAFT_REPO_ROOT
tag=$1; cfg=$2; st=$3; shift 3
mkdir -p gpurun_out
for v in "$@"; do
  lib=$v; [ $v = base ] && lib=
  PKV_LIB=$lib timeout 600 python bench.py --config $cfg --steps $st --warmup 5 --no-cpu --no-dense --no-1m > gpurun_out/var_${tag}_$v.log 2>&1
  echo "$v: $(python -c "
import json;d=json.loads(open('gpurun_out/var_${tag}_$v.log').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], {k: v['avg_us'] for k, v in d['kernels'].items()}, d.get('scan_hbm', {}).get('gbs'))" 2>&1 | tail -1)"
done

# usage: bash scripts/gpu_final.sh <tag> : round-end evidence — tests, contract bench line (CPU oracle baseline),
# reference arm, other configs (fp32 and fp16 weights), ncu --set full capture with DRAM traffic
cd $GRAFT_REPO_ROOT
tag=${1:-final}
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_$tag.log 2>&1; tail -2 gpurun_out/pytest_$tag.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_cpt_kernel|topk_cl_kernel" -s 10 -c 5 -o gpurun_out/prof_$tag python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense > gpurun_out/ncu_full_$tag.log 2>&1
ncu -i gpurun_out/prof_$tag.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_raw.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_${tag}_warm.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu --no-dense > /dev/null 2>&1
timeout 900 python bench.py --steps 200 --warmup 5 > gpurun_out/bench_${tag}_128k.log 2>&1; tail -c 300 gpurun_out/bench_${tag}_128k.log; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${tag}_ref.log 2>&1; tail -c 200 gpurun_out/bench_${tag}_ref.log; echo
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu --w16 > gpurun_out/bench_${tag}_128k_w16.log 2>&1
timeout 900 python bench.py --config 32k_bs8 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_${tag}_32k.log 2>&1
timeout 1200 python bench.py --config 1m --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_${tag}_1m.log 2>&1
timeout 1200 python bench.py --config 1m --steps 20 --warmup 3 --no-cpu --w16 > gpurun_out/bench_${tag}_1m_w16.log 2>&1
for f in 128k 128k_w16 32k 1m 1m_w16; do python -c "import json;d=json.loads(open('gpurun_out/bench_${tag}_$f.log').read().strip().splitlines()[-1]);print('$f', d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d.get('dense_sdpa_us_per_layer'))"; done
echo done

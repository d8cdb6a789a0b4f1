# usage: bash scripts/gpu_evidence.sh <tag> : round evidence — GPU tests, ncu --set full at 128K and 1M (+ raw
# csv for ncu_traffic.py), warm launch list, the contract bench line (with the CPU-oracle baseline), the
# reference arm and the variant lines (32K bs8, 1M, 1M --k-hbm, fp16 weights)
cd $GRAFT_REPO_ROOT
tag=${1:-ev}
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_$tag.log 2>&1; tail -2 gpurun_out/pytest_$tag.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_cpt_kernel|topk_cl_kernel" -s 10 -c 5 -o gpurun_out/prof_${tag}_128k python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense > gpurun_out/ncu_${tag}_128k.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"qprep_kernel|scan_kernel|select_kernel|rerank_cpt_kernel|topk_cl_kernel" -s 10 -c 5 -o gpurun_out/prof_${tag}_1m python bench.py --config 1m --layers 2 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense > gpurun_out/ncu_${tag}_1m.log 2>&1
for c in 128k 1m; do
  ncu -i gpurun_out/prof_${tag}_$c.ncu-rep --page raw --csv > gpurun_out/prof_${tag}_${c}_raw.csv 2>/dev/null
  python scripts/ncu_full_summary.py gpurun_out/prof_${tag}_$c.ncu-rep "ncu --set full --clock-control none, $c ($tag)" > gpurun_out/ncu_full_${tag}_$c.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_${tag}_warm.csv python bench.py --layers 2 --steps 2 --warmup 3 --no-cpu --no-dense > /dev/null 2>&1
timeout 900 python bench.py --steps 200 --warmup 5 > gpurun_out/bench_${tag}_128k.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${tag}_ref.log 2>&1
timeout 900 python bench.py --steps 200 --warmup 5 --no-cpu --w16 > gpurun_out/bench_${tag}_128k_w16.log 2>&1
timeout 900 python bench.py --config 32k_bs8 --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_${tag}_32k.log 2>&1
timeout 1200 python bench.py --config 1m --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_${tag}_1m.log 2>&1
timeout 1200 python bench.py --config 1m --steps 30 --warmup 5 --no-cpu --k-hbm > gpurun_out/bench_${tag}_1m_khbm.log 2>&1
for f in 128k 128k_w16 32k 1m 1m_khbm; do python -c "import json;d=json.loads(open('gpurun_out/bench_${tag}_$f.log').read().strip().splitlines()[-1]);print('$f', d['value'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['bound'], d['roofline']['frac'], d.get('dense_sdpa_us_per_layer'), d['clocks'])"; done
tail -c 400 gpurun_out/bench_${tag}_ref.log
echo done

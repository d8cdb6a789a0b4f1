# usage: bash scripts/evidence_collect.sh <tag> : copy one gpu_evidence.sh run from gpurun_out/ into profiles/r02/
#   (bench lines, phase anatomy, warm launch lists + medians, ncu --set full summaries, DRAM traffic)
tag=${1:-ev}
set -e
for f in 128k_with_1m 32k_bs8 128k_key_fraction 1m_khbm; do tail -1 gpurun_out/bench_${tag}_$f.log > profiles/r02/bench_$f.json; done
cp gpurun_out/phase_${tag}_128k.txt profiles/r02/phase_128k.txt
cp gpurun_out/phase_${tag}_1m.txt profiles/r02/phase_1m.txt
python scripts/ncu_warm_json.py profiles/r02/ncu_warm.json 128k=gpurun_out/launches_128k_$tag.csv 1m=gpurun_out/launches_1m_$tag.csv > /dev/null
python scripts/ncu_traffic.py gpurun_out/full_128k_${tag}_raw.csv 128k profiles/r02/ncu_traffic.json > /dev/null
python scripts/ncu_traffic.py gpurun_out/full_1m_${tag}_raw.csv 1m profiles/r02/ncu_traffic.json > /dev/null
python scripts/ncu_full_summary.py gpurun_out/full_128k_$tag.ncu-rep "ncu --set full, one layer at 128K" > profiles/r02/ncu_full_128k.txt
python scripts/ncu_full_summary.py gpurun_out/full_1m_$tag.ncu-rep "ncu --set full, one layer at 1M" > profiles/r02/ncu_full_1m.txt
for c in 128k 1m; do
python - "$c" "$tag" <<'PY'
import csv, sys
c, tag = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{c}_{tag}.csv")) if len(r) > 14 and r[0].isdigit()]
with open(f"profiles/r02/ncu_launches_{c}.csv", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none (warm, serialised), "
            f"python bench.py --config {c} --steps 1 --warmup 3 --layers 4 --no-cpu --no-dense --no-1m\n")
    f.write("id,kernel,grid,block,duration,unit\n")
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")[-60:]
        f.write(f"{r[0]},{name},\"{r[8]}\",\"{r[7]}\",{r[14]},{r[13]}\n")
PY
done
for f in 128k_with_1m 32k_bs8 128k_key_fraction 1m_khbm; do python -c "
import json;d=json.load(open('profiles/r02/bench_$f.json'));m=d.get('configs',{}).get('1m')
print('$f', d['value'], d['e2e']['value'], d.get('dense_sdpa_us_per_layer'), d['roofline']['kernel'], d['roofline']['frac'], 'enc', d.get('encode_us_per_layer'), '1m', m and m['value'], m and m['e2e']['value'])"; done
python -c "
import json;d=json.load(open('profiles/r02/ncu_warm.json'))
for c in d: print(c, d[c]['kernels_median_us'])"

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_drift_gpu.py -q 2>&1 | tail -2
timeout 1500 python scripts/drift_recall.py --prefill 32768 --decode 32768 --rates 0,0.0005,0.002 --out gpurun_out/drift_recall_r01.json 2>&1 | tail -4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:encode_kernel -c 1 -o gpurun_out/prof_enc python bench.py --layers 1 --steps 1 --warmup 3 --no-cpu --no-graph --no-dense > /dev/null 2>&1
ncu -i gpurun_out/prof_enc.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|DRAM Throughput|Compute \(SM\) Throughput|Issued Warp Per Scheduler|Achieved Occupancy|Registers Per Thread|Executed Ipc Active)"' | awk -F'","' '{print $(NF-2)" | "$NF}'
ncu -i gpurun_out/prof_enc.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/prof_enc_raw.csv

cd $GRAFT_REPO_ROOT
python -m paper_2602_07721_b200.build > /dev/null 2>&1 || exit 1
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_stream_gpu.py -q -x 2>&1 | tail -1
for l in "" ""; do PKV_LIB=$l timeout 600 python bench.py --layers 4 --steps 20 --warmup 3 --no-cpu --no-dense > gpurun_out/enc_$l.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/enc_$l.log').read().strip().splitlines()[-1]);print('[$l]', d['encode_us_per_layer'], d['encode_gbs'], d['value'])"; done

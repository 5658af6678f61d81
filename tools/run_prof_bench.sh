# bench + ncu captures of the bench's own launches (ViT-H, batch 64): launch list, full sets
timeout 200 python -m pytest tests/test_gpu_encoder.py -q -x --timeout 120 2>&1 | tail -2
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], d['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"zs_gemm2|zs_attn_win|zs_attn_glob" -s 3 -c 6 \
    -o gpurun_out/bench_full -f python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo "full rc=$?"

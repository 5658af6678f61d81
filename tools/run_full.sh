# Full round measurement on one B200: gpu tests, smoke, bench (+dense, +cpu), reference arm,
# ncu launch list of the bench command, ncu --set full of the top kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-400
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/launches_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zs_gemm2 -s 4 -c 4 -o gpurun_out/gemm_full -f \
    python tools/gemm_prof.py 8 > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zs_attn -c 2 -o gpurun_out/attn_full -f \
    python tools/attn_prof.py both > /dev/null 2>&1; echo "ncu attn rc=$?"
ls -la gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"zs_gemm2|zs_attn_win|zs_attn_glob" -s 3 -c 6 \
    -o gpurun_out/bench_full -f python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu bench_full rc=$?"
ls -la gpurun_out
timeout 900 python tools/density_sweep.py 16 --out gpurun_out/density_sweep.json > gpurun_out/density_sweep.log 2>&1; echo "sweep rc=$?"

# Round-2 full measurement on one B200: GPU tests, smoke, bench (+dense, +cpu), reference arm,
# BASELINE configs 2/3, ncu launch list of one bench step, ncu --set full of the step's GEMM and
# attention launches.  Results under gpurun_out/ (copied to profiles/ by hand).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-200
rm -f gpurun_out/configs.jsonl; bash tools/run_configs.sh > gpurun_out/configs.log 2>&1; cat gpurun_out/configs.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > gpurun_out/launches_step.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"zs_gemm2|zs_attn_win|zs_attn_glob" -c 40 -o gpurun_out/step_full -f python tools/prof_step.py > gpurun_out/step_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out

# Round-2 final measurement on one B200 (small outputs only): GPU tests, smoke, default bench,
# reference arm, BASELINE configs 2/3 (with clocks), density sweep (config 5).
set -x
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; tail -1 $O/bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1; tail -1 $O/bench_ref.log | cut -c1-200
rm -f gpurun_out/configs.jsonl; bash tools/run_configs.sh > $O/configs.log 2>&1; cp gpurun_out/configs.jsonl $O/; cat $O/configs.log
timeout 900 python tools/density_sweep.py 16 --out $O/density_sweep.json > $O/density_sweep.log 2>&1; echo "sweep rc=$?"
du -sh gpurun_out

# scratch gpurun payload used for one-off checks during development (A/B runs, bisects); see the
# other run_*.sh scripts for the maintained measurement recipes
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 2>&1 | tail -2

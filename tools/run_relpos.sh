timeout 400 python -m pytest tests/test_gpu_relpos.py -q -x --timeout 200 2>&1 | tail -4

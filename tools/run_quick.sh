timeout 300 python -m pytest tests/test_gpu_relpos.py -q -x -k encoder --timeout 200 2>&1 | tail -4

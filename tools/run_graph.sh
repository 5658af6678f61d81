timeout 300 python -m pytest tests/test_gpu_encoder.py -q -x -k "graph" --timeout 200 2>&1 | tail -3
timeout 300 python tools/graph_latency.py vit_h 1 4 2>&1 | tail -3
timeout 300 python tools/graph_latency.py vit_b 1 2>&1 | tail -2

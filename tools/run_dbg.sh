timeout 120 python tools/sobel_ab.py
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -q -x -k "sobel or order or saliency" --timeout 120 2>&1 | tail -2

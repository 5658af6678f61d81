timeout 300 python tools/gemm_ab.py 48 fc1,fc1nogelu,proj,proj16,qkv 2>&1 | tail -5

timeout 300 python tools/attn_ab.py global 16 stripes 2>&1 | grep median

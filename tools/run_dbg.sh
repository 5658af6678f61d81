ZS_AB_LIBS=libzstripe_b200_old.so,libzstripe_b200_reg160.so timeout 300 python tools/attn_ab.py local 64 2>&1 | grep -A1 median

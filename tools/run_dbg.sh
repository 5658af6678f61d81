ZS_AB_LIBS=libzstripe_b200.so,libzstripe_b200_old.so,libzstripe_b200_p1.so,libzstripe_b200_p2.so,libzstripe_b200_p3.so timeout 300 python tools/attn_ab.py local 64 2>&1 | grep -A1 median

ZS_AB_LIBS=libzstripe_b200.so,libzstripe_b200_old.so,libzstripe_b200_lsuout.so,libzstripe_b200_skipout.so timeout 300 python tools/attn_ab.py local 64 2>&1 | grep -A1 median
ZS_AB_LIBS=libzstripe_b200.so,libzstripe_b200_old.so,libzstripe_b200_lsuout.so timeout 300 python tools/attn_ab.py local 64 rows 2>&1 | grep -A1 median

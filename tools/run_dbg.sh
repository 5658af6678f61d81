ZS_AB_LIBS=libzstripe_b200.so,libzstripe_b200_old.so,libzstripe_b200_halfbias.so timeout 300 python tools/attn_ab.py global 16 stripes 2>&1 | grep median

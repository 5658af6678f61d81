L=paper_2605_17633_b200/_lib
cp $L/libzstripe_b200.so /tmp/main.so
for v in lsu2 lsu3 lsu4; do
  cp $L/libzstripe_b200_$v.so $L/libzstripe_b200.so
  ZS_G2_TMA_ALL=1 timeout 60 python tools/g2_bisect.py 235200 1280 1280 inplace 2>&1 | tail -1
  ZS_G2_TMA_ALL=1 timeout 60 python tools/g2_bisect.py 192 256 256 inplace 2>&1 | tail -1
  cp /tmp/main.so $L/libzstripe_b200.so
  echo "== $v"
  ZS_G2_TMA_ALL=1 ZS_AB_NEW=libzstripe_b200_$v.so timeout 300 python tools/gemm_ab.py 48 proj,fc2 2>&1 | tail -2
done

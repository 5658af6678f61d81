# EPI 3 buffer / stage variants: correctness (bisect cases) + paired A/B vs the LSU epilogue (HEAD)
L=paper_2605_17633_b200/_lib
cp $L/libzstripe_b200.so /tmp/main.so
for v in main rb3s4 rb3s4l rb4s3 rb4s3l; do
  if [ $v != main ]; then cp $L/libzstripe_b200_$v.so $L/libzstripe_b200.so; fi
  for c in "192 256 256 inplace" "256 256 256 mod" "235200 1280 1280 inplace"; do
    timeout 60 python tools/g2_bisect.py $c 2>&1 | tail -1
  done
  cp /tmp/main.so $L/libzstripe_b200.so
  echo "== $v"
  if [ $v = main ]; then n=libzstripe_b200.so; else n=libzstripe_b200_$v.so; fi
  ZS_AB_NEW=$n timeout 300 python tools/gemm_ab.py 48 proj,fc2 2>&1 | tail -2
done

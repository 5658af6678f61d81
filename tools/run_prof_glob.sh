# ncu --set full of the global attention kernel (ViT-H shapes, 16 images); report -> gpurun_out/
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"zs_attn_glob" -s 1 -c 1 -o gpurun_out/attn_glob_${1:-r2} -f python tools/attn_bench.py global 16 prof > gpurun_out/prof_glob.log 2>&1; echo "rc=$?"

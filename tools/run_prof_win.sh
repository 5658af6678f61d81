# ncu --set full of the window attention kernel (ViT-H shapes, 64 images); report -> gpurun_out/
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"zs_attn_win" -s 1 -c 1 -o gpurun_out/attn_win_${1:-r2} -f python tools/attn_prof.py local 64 > gpurun_out/prof_win.log 2>&1; echo "rc=$?"

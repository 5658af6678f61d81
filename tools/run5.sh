set -x
timeout 600 ncu --set full --import-source on -k regex:zs_attn -s 1 -c 1 -o gpurun_out/attn_local python tools/attn_prof.py local > gpurun_out/ncu_local.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:zs_attn -s 1 -c 1 -o gpurun_out/attn_global python tools/attn_prof.py global > gpurun_out/ncu_global.log 2>&1
tail -5 gpurun_out/ncu_local.log gpurun_out/ncu_global.log
ls -la gpurun_out

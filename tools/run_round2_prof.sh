# Round-2 ncu evidence of the bench's own launches (tools/prof_step.py: one ViT-H batch-64 forward in a
# profiler region), summarised ON THE BOX so only small files come back:
#   launch list (every kernel, cold-cache serialised) -> round2_launches.json
#   ncu --set full of block 0's GEMMs, the first window and the first global attention launch
#   -> round2_ncu_full_step.json (+ stall-by-opcode text for the attention kernels)
mkdir -p gpurun_out/prof
cd gpurun_out/prof
R=$GRAFT_REPO_ROOT
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file launches.csv python $R/tools/prof_step.py > /dev/null 2>&1; echo "launches rc=$?"
python $R/tools/launch_share.py launches.csv --out round2_launches.json > /dev/null; echo "share rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zs_gemm2 -c 5 -o gemm -f python $R/tools/prof_step.py > /dev/null 2>&1; echo "gemm rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zs_attn_win -c 1 -o attn_win -f python $R/tools/prof_step.py > /dev/null 2>&1; echo "win rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:zs_attn_glob -c 1 -o attn_glob -f python $R/tools/prof_step.py > /dev/null 2>&1; echo "glob rc=$?"
python $R/tools/ncu_summary.py gemm.ncu-rep attn_win.ncu-rep attn_glob.ncu-rep --out round2_ncu_full_step.json > /dev/null; echo "summary rc=$?"
python $R/tools/ncu_stall_ops.py attn_win.ncu-rep zs_attn_win 1000 > round2_stalls_attn_win.txt 2>&1
python $R/tools/ncu_stall_ops.py attn_glob.ncu-rep zs_attn_glob 1000 > round2_stalls_attn_glob.txt 2>&1
ls -la
rm -f gemm.ncu-rep
du -sh .

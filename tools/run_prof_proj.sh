# ncu --set full of the proj GEMM (fp32 residual, LSU epilogue) alone; summaries written on the box
mkdir -p gpurun_out/projprof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"zs_gemm2_kernel" -s 5 -c 1 -o gpurun_out/projprof/proj -f python tools/gemm_prof.py 48 > gpurun_out/projprof/ncu.log 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/projprof/proj.ncu-rep --out gpurun_out/projprof/summary.json > /dev/null 2>&1
python tools/ncu_stall_ops.py gpurun_out/projprof/proj.ncu-rep zs_gemm2 > gpurun_out/projprof/stalls.txt 2>&1
ncu -i gpurun_out/projprof/proj.ncu-rep --page raw --csv > gpurun_out/projprof/raw.csv 2>&1
ncu -i gpurun_out/projprof/proj.ncu-rep --page source --csv --print-source=sass,cuda > gpurun_out/projprof/source.csv 2>&1
ls -la gpurun_out/projprof; du -sh gpurun_out

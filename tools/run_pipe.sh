mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_17633_b200/csrc tools/pipe_bench.cu -o /tmp/pipe_bench && /tmp/pipe_bench > gpurun_out/pipe_bench.txt 2>&1
cat gpurun_out/pipe_bench.txt
python tools/attn_bench.py global 16 2>&1 | tail -5

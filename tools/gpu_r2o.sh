# one-warp K2 at 12 warps per SM (168 registers, no spills in the loop with SST2) against 8; FP64 latency probes
mkdir -p gpurun_out/r2o
bash tools/gpu_ab_c3.sh main w12 | tee gpurun_out/r2o/ab.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/microbench tools/microbench.cu && /tmp/microbench | tee gpurun_out/r2o/microbench.txt

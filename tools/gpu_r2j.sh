# K2 one-warp loop variants on C3 (128 utterances): rotated loop, unroll 2
mkdir -p gpurun_out/r2j
bash tools/gpu_ab_c3.sh main rot rotu2 | tee gpurun_out/r2j/ab.txt

// fp64_rf_bench.cu -- FP64 pipe throughput vs register-operand pattern (B200).
// Each thread runs 8 independent chains a_k <- op(a_k, b?, c?) for ITERS steps.
//   shared : fma(a_k, b, c)          (b, c common -> operand reuse cache)
//   dist3  : fma(a_k, b_k, c_k)      (3 distinct 64-bit registers per DFMA)
//   dist2  : fma(a_k, b_k, a_k)      (2 distinct)
//   dmul2  : a_k * b_k               (DMUL, 2 distinct)
//   dadd2  : a_k + b_k
// Prints thread-instructions/clk/SM (peak 64 for the FP64 pipe).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
template <int MODE>
__global__ void __launch_bounds__(256) k(const double* in, double* out) {
  double a[8], b[8], c[8];
#pragma unroll
  const int o = threadIdx.x & 1;
  for (int i = 0; i < 8; ++i) { a[i] = in[i + o]; b[i] = in[8 + i + o]; c[i] = in[16 + i + o]; }
  const double bb = in[29 + o], cc = in[30 + o];
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fma(a[i], bb, cc);
      if (MODE == 1) a[i] = fma(a[i], b[i], c[i]);
      if (MODE == 2) a[i] = fma(a[i], b[i], a[i]);
      if (MODE == 3) a[i] = a[i] * b[i];
      if (MODE == 4) a[i] = a[i] + b[i];
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, const double* din, double* dout) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int dev; cudaGetDevice(&dev); int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int warps : {4, 8, 16}) {
    const int blocks = sms * warps * 32 / 256;
    k<MODE><<<blocks, 256>>>(din, dout);
    cudaEventRecord(e0);
    k<MODE><<<blocks, 256>>>(din, dout);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double inst = double(blocks) * 256 * ITERS * 8;
    // clocks: assume the SM clock reported by nvidia-smi at load (~1.965 GHz); print per-ns too
    printf("%-7s warps/SM=%2d  %.3f ms  %.1f thread-inst/ns/SM  (=%.1f /clk at 1.965 GHz)\n", name, warps, ms,
           inst / (ms * 1e6) / sms, inst / (ms * 1e6) / sms / 1.965);
  }
}
int main() {
  double h[32];
  for (int i = 0; i < 32; ++i) h[i] = 1.0 + 1e-9 * i;
  h[30] = 1.0000000001; h[31] = 1e-300;
  double *din, *dout; cudaMalloc(&din, 256); cudaMalloc(&dout, 256 * 8);
  cudaMemcpy(din, h, 256, cudaMemcpyHostToDevice);
  run<0>("shared", din, dout); run<1>("dist3", din, dout); run<2>("dist2", din, dout);
  run<3>("dmul2", din, dout); run<4>("dadd2", din, dout);
  return 0;
}

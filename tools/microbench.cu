// microbench.cu -- FP64 latency / throughput probes on the B200 used to shape
// k_accel (development tool; not part of the product library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, int n, double a, double b) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  out[0] = x;
  out[1] = double(t1 - t0) / n;
}
__global__ void lat_dmul(double* out, int n, double a, double b) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * b;
  long long t1 = clock64();
  out[0] = x;
  out[1] = double(t1 - t0) / n;
}
__global__ void lat_rcp(double* out, int n, double a) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r + 1.0;
  }
  long long t1 = clock64();
  out[0] = x;
  out[1] = double(t1 - t0) / n;
}
__global__ void lat_shfl(double* out, int n, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1] = double(t1 - t0) / n;
}
// throughput: ILP independent DFMA chains per thread, many warps
template <int ILP>
__global__ void tput(double* out, int n, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = a + k;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], b, a);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}

template <int ILP>
void run_tput(double* d, int warps_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4000, threads = 128, blocks = 148 * warps_per_sm / 4;
  tput<ILP><<<blocks, threads>>>(d, 100, 1.0, 0.999999);
  cudaEventRecord(e0);
  tput<ILP><<<blocks, threads>>>(d, n, 1.0, 0.999999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * ILP * double(n) * blocks * threads;
  printf("tput ILP=%d warps/SM=%2d: %6.2f TFLOP/s\n", ILP, warps_per_sm, flops / (ms * 1e-3) / 1e12);
}

int main1();
int main2();
int main3();
int main() { main3(); main2(); return main1(); }
int main1() {
  double* d;
  cudaMalloc(&d, 64 * sizeof(double));
  double h[2];
  lat_dfma<<<1, 1>>>(d, 10000, 1.0, 0.9999);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h[1]);
  lat_dmul<<<1, 1>>>(d, 10000, 1.0, 0.9999);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("DMUL dependent latency: %.2f cycles\n", h[1]);
  lat_rcp<<<1, 1>>>(d, 10000, 1.5);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("MUFU.RCP64H + DADD dependent latency: %.2f cycles\n", h[1]);
  lat_shfl<<<1, 32>>>(d, 10000, 1.0);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("SHFL(f64) + DADD dependent latency: %.2f cycles\n", h[1]);
  for (int w : {4, 8, 16, 32}) {
    run_tput<1>(d, w);
    run_tput<2>(d, w);
    run_tput<4>(d, w);
    run_tput<8>(d, w);
  }
  return 0;
}

// DMMA m8n8k4 f64 dependent latency (D feeds C of the next)
__global__ void lat_dmma(double* out, int n) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 1.0, c0 = 0.0, c1 = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  out[threadIdx.x] = c0 + c1;
  if (threadIdx.x == 0) out[1] = double(t1 - t0) / n;
}
// smem broadcast LDS.128 + DADD dependent latency
__global__ void lat_lds(double* out, int n) {
  __shared__ double2 s[64];
  if (threadIdx.x < 64) s[threadIdx.x] = make_double2(threadIdx.x, 1.0);
  __syncwarp();
  int idx = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double2 v = s[idx];
    acc += v.x;
    idx = int(v.y) & 63;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) out[1] = double(t1 - t0) / n;
}
__global__ void lat_bar(double* out, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1] = double(t1 - t0) / n;
}
int main2() {
  double* d;
  cudaMalloc(&d, 256 * sizeof(double));
  double h[2];
  lat_dmma<<<1, 32>>>(d, 10000);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("DMMA m8n8k4 dependent latency: %.2f cycles (%s)\n", h[1], cudaGetErrorString(cudaGetLastError()));
  lat_lds<<<1, 32>>>(d, 10000);
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("LDS.128 + DADD dependent latency: %.2f cycles\n", h[1]);
  for (int nt : {64, 128, 256}) {
    lat_bar<<<1, nt>>>(d, 10000);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("__syncthreads (%d threads, all arriving together): %.2f cycles\n", nt, h[1]);
  }
  return 0;
}

// accuracy of the MUFU.RCP64H seed and of 1 / 2 Newton refinements
__global__ void rcp_acc(double* out, int n) {
  double m0 = 0, m1 = 0, m2 = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = 1.0 + (double)i / n * 7.0 + 1e-9 * (i % 977);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    const double e = fma(-x, r, 1.0);
    m0 = fmax(m0, fabs(e));
    const double r1 = fma(r, e, r);
    m1 = fmax(m1, fabs(fma(-x, r1, 1.0)));
    const double r2 = fma(r, fma(e, e, e), r);
    m2 = fmax(m2, fabs(fma(-x, r2, 1.0)));
  }
  atomicMax((unsigned long long*)&out[0], __double_as_longlong(m0));
  atomicMax((unsigned long long*)&out[1], __double_as_longlong(m1));
  atomicMax((unsigned long long*)&out[2], __double_as_longlong(m2));
}
int main3() {
  double* d;
  cudaMalloc(&d, 4 * sizeof(double));
  cudaMemset(d, 0, 4 * sizeof(double));
  rcp_acc<<<148, 256>>>(d, 1 << 24);
  double h[3];
  cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("rcp seed max |1-x r| = %.3e (2^%.1f); one Newton: %.3e; Newton+cubic: %.3e\n", h[0], log2(h[0]), h[1], h[2]);
  return 0;
}

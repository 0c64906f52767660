// nan_probe.cu -- which NaN bit patterns do B200's FP64 / FP32 units produce?
// (development probe: K2's integer-compare floor keeps a NaN only if its sign
// bit is clear). Feeds quiet NaNs of both signs and NaN-producing operands
// through DFMA / DMUL / DADD / MUFU.RCP64H (and FP32 counterparts) with negate
// modifiers, and prints the result bits.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/nan_probe tools/nan_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(const double* in, unsigned long long* out, const float* fin, unsigned* fout) {
  const double p = in[0], n = in[1], one = in[2], inf = in[3], zero = in[4];
  int k = 0;
  auto put = [&](double v) { out[k++] = __double_as_longlong(v); };
  put(fma(p, one, one));      // +NaN * 1 + 1
  put(fma(-p, one, one));     // -(+NaN) * 1 + 1
  put(fma(n, one, one));      // -NaN * 1 + 1
  put(fma(one, -one, n));     // 1 * -1 + -NaN
  put(p * -one);
  put(n * one);
  put(-n + one);
  put(inf - inf);             // invalid operation
  put(zero * inf);
  put(fma(-one, zero * inf, one));
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(n));
  put(r);
  put(fma(-r, one, one));
  int j = 0;
  auto fput = [&](float v) { fout[j++] = __float_as_uint(v); };
  const float fp = fin[0], fn = fin[1], fo = fin[2];
  fput(fmaf(fp, fo, fo));
  fput(fmaf(-fp, fo, fo));
  fput(fmaf(fn, fo, fo));
  fput(fn * fo);
  fput(-fn + fo);
}

int main() {
  double h[5];
  unsigned long long pn = 0x7FF8000000000000ull, nn = 0xFFF8000000000001ull;
  memcpy(&h[0], &pn, 8); memcpy(&h[1], &nn, 8); h[2] = 1.0; h[3] = __builtin_inf(); h[4] = 0.0;
  float fh[3]; unsigned fpn = 0x7FC00000u, fnn = 0xFFC00001u;
  memcpy(&fh[0], &fpn, 4); memcpy(&fh[1], &fnn, 4); fh[2] = 1.0f;
  double* d; unsigned long long* o; float* fd; unsigned* fo;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 16 * 8); cudaMalloc(&fd, sizeof(fh)); cudaMalloc(&fo, 16 * 4);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpy(fd, fh, sizeof(fh), cudaMemcpyHostToDevice);
  k<<<1, 1>>>(d, o, fd, fo);
  unsigned long long r[12]; unsigned fr[5];
  cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  cudaMemcpy(fr, fo, sizeof(fr), cudaMemcpyDeviceToHost);
  const char* names[12] = {"fma(+nan,1,1)", "fma(-(+nan),1,1)", "fma(-nan,1,1)", "fma(1,-1,-nan)", "+nan*-1",
                           "-nan*1", "-(-nan)+1", "inf-inf", "0*inf", "fma(-1,0*inf,1)", "rcp(-nan)", "fma(-rcp,1,1)"};
  for (int i = 0; i < 12; ++i) printf("f64 %-18s %016llx %s\n", names[i], r[i], (r[i] >> 63) ? "NEGATIVE" : "positive");
  const char* fnames[5] = {"fmaf(+nan,1,1)", "fmaf(-(+nan),1,1)", "fmaf(-nan,1,1)", "-nan*1", "-(-nan)+1"};
  for (int i = 0; i < 5; ++i) printf("f32 %-18s %08x %s\n", fnames[i], fr[i], (fr[i] >> 31) ? "NEGATIVE" : "positive");
  return 0;
}

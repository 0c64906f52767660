// k2_cluster_probe.cu -- per-phase latency probe of the CLUSTER K2 (development
// tool, not part of the library). Builds k_accel with RCSCM_K2_PROBE for the
// config-4 shape (M = 8, J = 4096: 2-CTA clusters x 256 threads x 8 slots) and
// the config-2 shape (J = 20000: 16 x 256 x 5), constants in shared memory, on
// random well-posed per-slot inputs, and prints the mean cycles of each phase
// of iterations 4..14 (warp 0 of every CTA):
//   0->1 phase 1 (gamma, residual, lambda terms, in-thread tree)
//   1->2 warp total (DMMA)     2->3 phase 2 + __syncthreads
//   3->4 block total + cluster exchange (push, arrive, wait on the peers)
//   4->5 1/lambda + phase 3    5->0' loop back
// and the iteration-start offsets of the CTAs sharing an SM.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DRCSCM_K2_PROBE
//        -I paper_1908_01964_b200/csrc -o build/k2_cluster_probe tools/k2_cluster_probe.cu
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#ifndef RCSCM_K2_LB_THREADS
#define RCSCM_K2_LB_THREADS 256
#endif
#include "accel.cuh"

using namespace rcscm;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int SPT, int CL, int SMEMC = 1, int MINB = 0>
void run(const char* name, int nb, int J, int nt, int iters) {
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  const size_t S = static_cast<size_t>(nb) * J;
  std::vector<double2> sab(nb), sbx(S), tax(S);
  std::vector<double> taa(nb), txx(S), rh(S, 1.0), ru(S, 1.0), lam(nb, 1.0);
  for (int i = 0; i < nb; ++i) { sab[i] = make_double2(0.3 + 0.1 * nd(rng), 0.2); taa[i] = 1.0; }
  for (size_t s = 0; s < S; ++s) {
    sbx[s] = make_double2(nd(rng), nd(rng));
    tax[s] = make_double2(nd(rng), nd(rng));
    txx[s] = 3.0 + std::abs(nd(rng));
  }
  auto up = [](const void* h, size_t n) { void* d; CK(cudaMalloc(&d, n)); CK(cudaMemcpy(d, h, n, cudaMemcpyHostToDevice)); return d; };
  AccelArgs A = {};
  A.nb = nb; A.J = J; A.iters = iters; A.inv_M = 0.125; A.k1 = 0.5; A.k2 = 0.0; A.eps = 1e-10; A.gamma_fault = 0.0;
  A.sigma_ab = (const double2*)up(sab.data(), nb * 16);
  A.tau_aa = (const double*)up(taa.data(), nb * 8);
  A.sigma_bx = (const double2*)up(sbx.data(), S * 16);
  A.tau_ax = (const double2*)up(tax.data(), S * 16);
  A.tau_xx = (const double*)up(txx.data(), S * 8);
  A.r_h_in = (const double*)up(rh.data(), S * 8);
  A.r_u_in = (const double*)up(ru.data(), S * 8);
  A.lambda_in = (const double*)up(lam.data(), nb * 8);
  CK(cudaMalloc(&A.r_h, S * 8)); CK(cudaMalloc(&A.r_u, S * 8)); CK(cudaMalloc(&A.lambda, nb * 8));
  const int ncta = nb * CL;
  long long* dprobe;
  const size_t np = static_cast<size_t>(ncta) * 8 * 16 * 8;
  CK(cudaMalloc(&dprobe, np * 8));
  CK(cudaMemset(dprobe, 0, np * 8));
  CK(cudaMemcpyToSymbol(g_k2_probe, &dprobe, sizeof(dprobe)));
  const bool full = (static_cast<long long>(nt) * SPT * CL == J);
  auto kern = full ? k_accel<SPT, CL, true, false, SMEMC, MINB, true, double> : k_accel<SPT, CL, false, false, SMEMC, MINB, true, double>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ncta);
  cfg.blockDim = dim3(nt);
  cfg.dynamicSmemBytes = SMEMC ? static_cast<size_t>(SPT) * nt * (SMEMC == 1 ? 6 : 4) * sizeof(double) : 0;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(cfg.dynamicSmemBytes)));
  if (CL > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.numAttrs = 1;
  cfg.attrs = attr;
  int nclusters = 0;
  CK(cudaOccupancyMaxActiveClusters(&nclusters, (void*)kern, &cfg));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) CK(cudaLaunchKernelEx(&cfg, kern, A));
  cudaEventRecord(e0);
  CK(cudaLaunchKernelEx(&cfg, kern, A));
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  std::vector<long long> h(np);
  CK(cudaMemcpy(h.data(), dprobe, np * 8, cudaMemcpyDeviceToHost));
  double acc[6] = {}; long cnt = 0;
  for (int b = 0; b < ncta; ++b)
    for (int w = 0; w < 1; ++w)
      for (int it = 4; it < 15; ++it) {
        const long long* p = &h[((static_cast<size_t>(b) * 8 + w) * 16 + it) * 8];
        const long long* q = &h[((static_cast<size_t>(b) * 8 + w) * 16 + it + 1) * 8];
        if (p[0] == 0 || q[0] == 0) continue;
        for (int k = 0; k < 5; ++k) acc[k] += static_cast<double>(p[k + 1] - p[k]);
        acc[5] += static_cast<double>(q[0] - p[5]);
        ++cnt;
      }
  double tot = 0;
  for (double& a : acc) { a /= cnt; tot += a; }
  printf("%s smemc=%d minb=%d nb=%d CL=%d nt=%d spt=%d active clusters %d: %.4f ms | ph1 %.0f | warp-red %.0f | ph2+bar %.0f | "
         "blk+exchange %.0f | rcp+ph3 %.0f | loop %.0f | iter %.0f cyc\n",
         name, SMEMC, MINB, nb, CL, nt, SPT, nclusters, ms, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], tot);
  // iteration-start offsets of the CTAs sharing an SM (warp 0, iterations 4..9)
  std::vector<std::vector<int>> by_sm(1024);
  for (int b = 0; b < ncta; ++b) {
    const long long smid = h[((static_cast<size_t>(b) * 8) * 16) * 8 + 7];
    if (h[((static_cast<size_t>(b) * 8) * 16 + 4) * 8] != 0) by_sm[smid & 1023].push_back(b);
  }
  int shown = 0;
  for (int sm = 0; sm < 1024 && shown < 4; ++sm) {
    if (by_sm[sm].size() < 2) continue;
    ++shown;
    printf("  sm %d:", sm);
    const long long t00 = h[((static_cast<size_t>(by_sm[sm][0]) * 8) * 16 + 4) * 8];
    for (int b : by_sm[sm]) {
      if (shown > 2 && b != by_sm[sm][0] && b != by_sm[sm][1]) continue;
      printf(" [cta %d:", b);
      for (int it = 4; it < 10; ++it) printf(" %lld", h[((static_cast<size_t>(b) * 8) * 16 + it) * 8] - t00);
      printf("]");
    }
    printf("\n");
  }
  cudaFree(dprobe);
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0 || which == 1) {
    // config 4 shape: M = 8, J = 4096
    run<8, 2>("c4 2x256x8", 2049, 4096, 256, 100);
    run<4, 4, 1, 4>("c4 4x256x4 minb4", 2049, 4096, 256, 100);
    run<8, 2, 2>("c4 2x256x8 smemc2", 2049, 4096, 256, 100);
    run<2, 8, 1, 4>("c4 8x256x2 minb4", 2049, 4096, 256, 100);
  }
  if (which == 3) {
    run<8, 2>("c4 2x256x8", 2049, 4096, 256, 100);
    run<8, 3>("c4 3x192x8", 2049, 4096, 192, 100);
    run<6, 3>("c4 3x256x6", 2049, 4096, 256, 100);
    run<6, 3, 1, 3>("c4 3x256x6 minb3", 2049, 4096, 256, 100);
    run<8, 4>("c4 4x128x8", 2049, 4096, 128, 100);
    run<4, 4, 1, 3>("c4 4x256x4 minb3", 2049, 4096, 256, 100);
  }
  if (which == 0 || which == 2) {
    // config 2 shape: J = 20000
    run<8, 16>("c2 16x160x8", 513, 20000, 160, 50);
    run<8, 10>("c2 10x256x8", 513, 20000, 256, 50);
    run<8, 12>("c2 12x224x8", 513, 20000, 224, 50);
    run<5, 16>("c2 16x256x5", 513, 20000, 256, 50);
  }
  return 0;
}

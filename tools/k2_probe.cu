// k2_probe.cu -- per-phase latency probe of K2 (development tool, not part of the
// library). Builds k_accel with RCSCM_K2_PROBE, runs nb bins x J = 640 on
// random, well-posed per-slot inputs (bin count chosen so 1, 2 or 3 CTAs share
// an SM), and prints the mean cycles of each phase of iterations 4..15:
//   0->1 phase 1 (gamma, residual, lambda terms, in-thread tree)
//   1->2 warp total (DMMA)     2->3 phase 2 + __syncthreads
//   3->4 block total + scale   4->5 1/lambda + phase 3     5->0' loop back
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DRCSCM_K2_PROBE
//        -I paper_1908_01964_b200/csrc -o build/k2_probe tools/k2_probe.cu
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "accel.cuh"

using namespace rcscm;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

int main(int argc, char** argv) {
  const int J = 640, iters = 100;
#ifdef RCSCM_K2_STAGGER
  for (long long st : {0LL, 150LL, 300LL, 500LL, 800LL})
#else
  for (long long st : {0LL})
#endif
  for (int nb : {148, 444, 1025}) {
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
    A.nb = nb; A.J = J; A.iters = iters; A.inv_M = 0.25; A.k1 = 0.5; A.k2 = 0.0; A.eps = 1e-10; A.gamma_fault = 0.0;
    A.sigma_ab = (const double2*)up(sab.data(), nb * 16);
    A.tau_aa = (const double*)up(taa.data(), nb * 8);
    A.sigma_bx = (const double2*)up(sbx.data(), S * 16);
    A.tau_ax = (const double2*)up(tax.data(), S * 16);
    A.tau_xx = (const double*)up(txx.data(), S * 8);
    A.r_h_in = (const double*)up(rh.data(), S * 8);
    A.r_u_in = (const double*)up(ru.data(), S * 8);
    A.lambda_in = (const double*)up(lam.data(), nb * 8);
    CK(cudaMalloc(&A.r_h, S * 8)); CK(cudaMalloc(&A.r_u, S * 8)); CK(cudaMalloc(&A.lambda, nb * 8));
    long long* dprobe;
    const size_t np = static_cast<size_t>(nb) * 8 * 16 * 8;
    CK(cudaMalloc(&dprobe, np * 8));
    CK(cudaMemset(dprobe, 0, np * 8));
#ifdef RCSCM_K2_PROBE
    CK(cudaMemcpyToSymbol(g_k2_probe, &dprobe, sizeof(dprobe)));
#endif
#ifndef K2_SPT
#define K2_SPT 5
#define K2_MINB 3
#endif
#ifndef K2_SMEMC
#define K2_SMEMC 0
#endif
    const int nt = J / K2_SPT;
    auto kern = k_accel<K2_SPT, 1, true, false, K2_SMEMC, K2_MINB, true, double>;
    const size_t dsm = K2_SMEMC ? static_cast<size_t>(K2_SPT) * nt * (K2_SMEMC == 1 ? 6 : 4) * sizeof(double) : 0;
    if (dsm) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dsm)));
#ifdef RCSCM_K2_STAGGER
    CK(cudaMemcpyToSymbol(g_k2_stagger, &st, sizeof(st)));
    std::vector<unsigned> zero(256, 0);
#endif
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int r = 0; r < 3; ++r) kern<<<nb, nt, dsm>>>(A);
#ifdef RCSCM_K2_STAGGER
    CK(cudaMemcpyToSymbol(g_k2_smcount, zero.data(), 256 * sizeof(unsigned)));
#endif
    cudaEventRecord(e0);
    kern<<<nb, nt, dsm>>>(A);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> h(np);
    CK(cudaMemcpy(h.data(), dprobe, np * 8, cudaMemcpyDeviceToHost));
    double acc[6] = {}; long cnt = 0;
    for (int b = 0; b < nb; ++b)
      for (int w = 0; w < 4; ++w)
        for (int it = 4; it < 15; ++it) {
          const long long* p = &h[((static_cast<size_t>(b) * 8 + w) * 16 + it) * 8];
          const long long* q = &h[((static_cast<size_t>(b) * 8 + w) * 16 + it + 1) * 8];
          for (int k = 0; k < 5; ++k) acc[k] += static_cast<double>(p[k + 1] - p[k]);
          acc[5] += static_cast<double>(q[0] - p[5]);
          ++cnt;
        }
    // phase relation of the CTAs sharing an SM: iteration-start stamps of warp 0
    {
      std::vector<std::vector<int>> by_sm(1024);
      for (int b = 0; b < nb; ++b) by_sm[h[((static_cast<size_t>(b) * 8) * 16) * 8 + 7] & 1023].push_back(b);
      int shown = 0;
      for (int sm = 0; sm < 1024 && shown < 3; ++sm) {
        if (by_sm[sm].size() < 2) continue;
        ++shown;
        printf("  sm %d:", sm);
        const long long t00 = h[((static_cast<size_t>(by_sm[sm][0]) * 8) * 16 + 4) * 8];
        for (int b : by_sm[sm]) {
          printf(" [cta %d:", b);
          for (int it = 4; it < 10; ++it) printf(" %lld", h[((static_cast<size_t>(b) * 8) * 16 + it) * 8] - t00);
          printf("]");
        }
        printf("\n");
      }
    }
    double tot = 0;
    for (double& a : acc) { a /= cnt; tot += a; }
#ifdef RCSCM_K2_STAGGER
    printf("stagger %lld nb=%4d %.4f ms\n", st, nb, ms);
    continue;
#endif
    printf("nb=%4d (%.2f CTA/SM) %.4f ms | ph1 %.0f | warp-red %.0f | ph2+bar %.0f | blk+scale %.0f | rcp+ph3 %.0f | loop %.0f | iter %.0f cyc\n",
           nb, nb / 148.0, ms, acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], tot);
  }
  return 0;
}

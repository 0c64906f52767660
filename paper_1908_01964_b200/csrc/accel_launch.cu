// accel_launch.cu -- K2 configuration choice and dispatch.
#include <cstdlib>

#include "accel_launch.cuh"

#ifndef RCSCM_K2_W1_MIN_BINS
#define RCSCM_K2_W1_MIN_BINS 2048  // one-warp CTAs from this many bins on (0: never)
#endif

namespace rcscm {

AccelCfg choose_accel_cfg(int64_t J, bool f32) {
  AccelCfg best{0, 0, 0, false, 0, 0, false, f32};
  const char* e_dir = std::getenv("RCSCM_ACCEL_DIRECT");
  const bool direct = e_dir ? std::atoi(e_dir) != 0 : true;  // measured faster (B200)
  const char* e_spt = std::getenv("RCSCM_ACCEL_SPT");
  const char* e_cl = std::getenv("RCSCM_ACCEL_CL");
  const char* e_sm = std::getenv("RCSCM_ACCEL_SMEM");
  // -1: per-configuration default (shared-memory constants for clusters of 4+, where
  // the cluster barrier needs more resident CTAs to hide; measured on B200)
  const int smem_env = e_sm ? std::atoi(e_sm) : -1;
  // MINB: CTAs per SM the 128-thread launch bounds target (0 = 256-thread bounds);
  // RCSCM_K2_MINB1 (launch.h) for register-resident constants (measured on B200)
  const char* e_mb = std::getenv("RCSCM_ACCEL_MINB");
  const int minb_env = e_mb ? std::atoi(e_mb) : -1;
  const int force_spt = e_spt ? std::atoi(e_spt) : 0;
  const int force_cl = e_cl ? std::atoi(e_cl) : 0;
  // the fewest CTAs per bin that hold it: clusters are bound by their per-
  // iteration exchange, which costs more with every CTA (measured on B200,
  // J = 20000: 10 x 256 x 8 2.26 ms against 16 x 160 x 8 2.64 ms and 12 x 224 x 8
  // 2.70 ms, tools/k2_cluster_probe.cu)
  for (int cl : {1, 2, 3, 4, 5, 6, 8, 10, 12, 16}) {
    if (force_cl && cl != force_cl) continue;
    const int64_t jc = (J + cl - 1) / cl;
    // FP32 state takes half the registers; clusters are bound by the per-iteration
    // DSMEM exchange, so the fewest CTAs per bin win (measured on B200: J = 4096
    // runs 33 % faster as 2 CTAs x 8 slots/thread than as 4 x 4)
    const int max_spt = (cl >= 2 || f32) ? 8 : 6;
    if (jc > 256LL * (force_spt ? force_spt : max_spt)) continue;
    // complex64 clusters (constants always in registers): CTAs of <= 128 threads,
    // so two CTAs of different clusters share an SM (measured on B200, config 4
    // c64: 4 x 128 x 8 2.18 ms against 2 x 256 x 8 2.35 ms)
    if (f32 && !force_cl && cl >= 2 && cl < 16 && jc > 128LL * max_spt) continue;
    int64_t best_waste = -1;
    for (int spt = 1; spt <= 8; ++spt) {
      if (spt == 7 || (cl >= 2 && spt < 4)) continue;  // not instantiated (accel_launch.cuh)
      if (force_spt ? spt != force_spt : spt > max_spt) continue;
      int64_t nt = (jc + spt - 1) / spt;
      nt = (nt + 31) / 32 * 32;
      if (nt > 256) continue;
      const int64_t waste = nt * spt - jc;
      // least idle lanes; ties go to more slots per thread (ILP, fewer warps)
      if (best_waste < 0 || waste < best_waste || (waste == best_waste && spt > best.spt)) {
        best_waste = waste;
        // FULL needs every CTA of the cluster to own exactly nt * spt frames
        const bool full = (waste == 0) && (jc * cl == J);
        // constants in registers everywhere: with the scalar carried state
        // (k_accel SST) a slot is 12 registers, so 8 slots fit the 128 that two
        // 256-thread CTAs per SM leave (measured on B200, against shared-memory
        // constants: C4 2.37 -> 2.24 ms, C2 1.78 -> 1.72 ms). Before SST a slot
        // took 20 registers and clusters kept their constants in shared memory.
        const int smem = smem_env >= 0 ? smem_env : 0;
        const int minb = minb_env >= 0 ? minb_env : (smem == 0 ? RCSCM_K2_MINB1 : 4);
        // complex64: shared-memory constants only for clusters of 8+ (instantiated
        // there; measured on B200, config 2 c64 as 16 x 160 x 8: 2.17 ms against
        // 4.40 ms with the constants in registers)
        const int smem_t = f32 ? (cl >= 8 ? (smem_env >= 0 ? smem_env : 1) : 0) : smem;
        // clusters always take the direct form (the affine one is single-CTA only)
        best = AccelCfg{cl, static_cast<int>(nt), spt, full, smem_t, minb, direct || cl >= 2, f32};
      }
    }
    if (best.cl) return best;
  }
  return best;
}

bool accel_fusable(const AccelCfg& g, int M) {
  const char* e = std::getenv("RCSCM_FUSE_PRE");
  if (e && std::atoi(e) == 0) return false;
  if (!(M == 2 || M == 4 || M == 8) || g.f32 || !g.direct) return false;
  // the tuned single-CTA shape, or a cluster with its constants in registers
  return (g.cl == 1 && g.full && g.smem == 0 && g.minb == RCSCM_K2_MINB1 && g.nt <= 128) || (g.cl >= 2 && g.smem == 0);
}

void accel_one_warp(AccelCfg& g, int64_t nb) {
  const char* e = std::getenv("RCSCM_ACCEL_W1");
  const int64_t min_nb = e ? std::atoll(e) : RCSCM_K2_W1_MIN_BINS;
  if (min_nb <= 0 || nb < min_nb) return;
  if (!g.prem || g.cl != 1 || !g.full || g.smem != 0 || g.nt != 64 || g.spt != 5 || g.we) return;
  g.we = 2;
  g.nt = 32;
  g.spt = 10;
}

cudaError_t launch_accel(cudaStream_t s, const AccelArgs& A, const AccelCfg& g) {
  if (A.nb * A.J == 0) return cudaSuccess;
  if (g.prem && g.cl == 1) return launch_accel_fused(s, A, g);
  switch (g.cl) {
    case 1: return launch_accel_cl1(s, A, g);
    case 2: return launch_accel_cl2(s, A, g);
    case 3: return launch_accel_cl3(s, A, g);
    case 4: return launch_accel_cl4(s, A, g);
    case 5: return launch_accel_cl5(s, A, g);
    case 6: return launch_accel_cl6(s, A, g);
    case 8: return launch_accel_cl8(s, A, g);
    case 10: return launch_accel_cl10(s, A, g);
    case 12: return launch_accel_cl12(s, A, g);
    case 16: return launch_accel_cl16(s, A, g);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace rcscm

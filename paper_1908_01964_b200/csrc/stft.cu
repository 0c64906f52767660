// stft.cu -- STFT analysis / WOLA synthesis on the GPU (the steps before and
// after the SCM path), sm_100a.
//
// Reference: stft.hpp:12-29 (periodic Hamming, WOLA dual window), :50-88
// (stft_analyze), :92-129 (stft_synthesize). The transforms are batched cuFFT
// D2Z / Z2D of length win over all (frame, channel) pairs; framing, windowing,
// the layout change to the Spectrogram layout ([bin][frame][mic]) and the
// overlap-add are our kernels. Batch order r = j*M + ch makes the spectrum a
// (J*M) x bins matrix whose transpose is exactly the [bin][frame][mic] layout,
// so one tiled transpose moves it. The overlap-add gathers, for every output
// sample, the frames covering it in ascending frame order -- the reference's
// accumulation order -- so no atomics are needed and results are deterministic.
#include <cufft.h>

#include "launch.h"

namespace rcscm {

// F[(j*M + ch)*win + k] = x(ch, j*hop - pad + k) * w[k] (0 outside [0, len));
// x(ch, p) at ch + p*M (Waveform::samples, M x len col-major) or, planar, at
// ch*len + p (one contiguous row per channel)
__global__ void k_stft_frames(const double* __restrict__ x, int64_t len, int M, int win, int hop, int64_t J,
                              const double* __restrict__ w, double* __restrict__ F, bool planar) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = blockIdx.y;
  if (k >= win || r >= J * M) return;
  const int64_t j = r / M, ch = r % M;
  const int64_t p = j * hop - (win - hop) + k;
  F[r * win + k] = (p >= 0 && p < len) ? x[planar ? ch * len + p : ch + p * M] * w[k] : 0.0;
}

// Half-spectrum input of the inverse transform: the imaginary parts of DC and
// (for even win) Nyquist are discarded, as the reference's real inverse FFT
// (Eigen FFT, HalfSpectrum) does.
__global__ void k_stft_clear_edges(double2* Z, int64_t rows, int64_t B, bool nyquist) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  Z[r * B].y = 0.0;
  if (nyquist) Z[r * B + B - 1].y = 0.0;
}

// out(ch, p) = sum over frames j covering p (ascending) of
//   F[(j*M + ch)*win + k] * (dual[k] / win),  k = p - (j*hop - pad)
// (stft.hpp:118-125; the 1/win is the inverse DFT's normalisation, exact for
// power-of-two win, folded into the dual-window table on the host).
__global__ void k_stft_ola(const double* __restrict__ F, int64_t len, int M, int win, int hop, int64_t J,
                           const double* __restrict__ dual_n, double* __restrict__ out, bool planar) {
  const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;  // ch + p*M, or ch*len + p
  if (q >= len * M) return;
  const int64_t p = planar ? q % len : q / M, ch = planar ? q / len : q % M;
  const int64_t pad = win - hop;
  // frames j with j*hop - pad <= p < j*hop - pad + win
  int64_t j0 = p + pad - win + 1;
  j0 = j0 <= 0 ? 0 : (j0 + hop - 1) / hop;
  int64_t j1 = (p + pad) / hop;
  if (j1 > J - 1) j1 = J - 1;
  double acc = 0.0;
  for (int64_t j = j0; j <= j1; ++j) {
    const int64_t k = p - (j * hop - pad);
    acc += F[(j * M + ch) * win + k] * dual_n[k];
  }
  out[q] = acc;
}

namespace {
cudaError_t cufft_status(cufftResult r) { return r == CUFFT_SUCCESS ? cudaSuccess : cudaErrorUnknown; }
}  // namespace

StftPlan::~StftPlan() { reset(); }
void StftPlan::reset() {
  if (fwd) cufftDestroy(static_cast<cufftHandle>(fwd));
  if (inv) cufftDestroy(static_cast<cufftHandle>(inv));
  fwd = inv = 0;
  n = 0;
  batch = 0;
}
cudaError_t StftPlan::ensure(int win, int64_t b, cudaStream_t s) {
  if (win == n && b == batch && fwd && inv) {
    cufftSetStream(static_cast<cufftHandle>(fwd), s);
    cufftSetStream(static_cast<cufftHandle>(inv), s);
    return cudaSuccess;
  }
  reset();
  const int bins = win / 2 + 1;
  int nn[1] = {win};
  cufftHandle f = 0, i = 0;
  cufftResult r = cufftPlanMany(&f, 1, nn, nn, 1, win, nn, 1, bins, CUFFT_D2Z, static_cast<int>(b));
  if (r != CUFFT_SUCCESS) return cufft_status(r);
  r = cufftPlanMany(&i, 1, nn, nn, 1, bins, nn, 1, win, CUFFT_Z2D, static_cast<int>(b));
  if (r != CUFFT_SUCCESS) {
    cufftDestroy(f);
    return cufft_status(r);
  }
  fwd = static_cast<int>(f);
  inv = static_cast<int>(i);
  n = win;
  batch = b;
  cufftSetStream(f, s);
  cufftSetStream(i, s);
  return cudaSuccess;
}

cudaError_t launch_stft_analyze(cudaStream_t s, StftPlan& plan, const double* x, int64_t len, int M, int win,
                                int hop, int64_t J, const double* window, double* frames, double2* spec,
                                double2* X, bool planar) {
  const int64_t rows = J * M, B = win / 2 + 1;
  if (rows == 0) return cudaSuccess;
  cudaError_t e = plan.ensure(win, rows, s);
  if (e != cudaSuccess) return e;
  k_stft_frames<<<dim3((win + 255) / 256, static_cast<unsigned>(rows)), 256, 0, s>>>(x, len, M, win, hop, J, window,
                                                                                  frames, planar);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  e = cufft_status(cufftExecD2Z(static_cast<cufftHandle>(plan.fwd), frames, reinterpret_cast<cufftDoubleComplex*>(spec)));
  if (e != cudaSuccess) return e;
  // spec: element (i, r) at i + r*B  ->  X[i*(J*M) + r] = X[(i*J + j)*M + ch]
  return launch_transpose_c(s, spec, X, B, rows, B, true);
}

cudaError_t launch_stft_synthesize(cudaStream_t s, StftPlan& plan, const double2* X, int64_t B, int64_t J, int M,
                                   int win, int hop, int64_t len, const double* dual_n, double2* spec,
                                   double* frames, double* out, bool planar) {
  const int64_t rows = J * M;
  if (len * M == 0) return cudaSuccess;
  cudaError_t e = plan.ensure(win, rows, s);
  if (e != cudaSuccess) return e;
  if ((e = launch_transpose_c(s, X, spec, B, rows, B, false)) != cudaSuccess) return e;
  k_stft_clear_edges<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(spec, rows, B, win % 2 == 0);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  e = cufft_status(cufftExecZ2D(static_cast<cufftHandle>(plan.inv), reinterpret_cast<cufftDoubleComplex*>(spec), frames));
  if (e != cudaSuccess) return e;
  k_stft_ola<<<static_cast<unsigned>((len * M + 255) / 256), 256, 0, s>>>(frames, len, M, win, hop, J, dual_n, out, planar);
  return cudaGetLastError();
}

}  // namespace rcscm

// traj_kernel.cu — NEXT row f1 of SURVEY.md §8(f): a moving source recorded by a microphone array
// (§3.4; library function of P:276).
//
//   out[m][t] = sum_j sig[j] rir[p(j)][m][t - j],   0 <= t - j < L,   0 <= t < n_sig + L - 1,
//   p(j) = min(j / floor(n_sig / n_points), n_points - 1)   (contiguous segments, reading R7 = SPEC S:414).
//
// The paper overlap-adds FFT products (cuFFT + a pointwise kernel).  Here the same linear filter is a
// direct time-domain convolution: on B200 the RIR-length x signal-length MACs of a dataset's trajectories
// are a few GFLOP, FFMA-bound, exact in fp32 and deterministic (no FFT round-off, fixed summation
// order).  One CTA computes kCvTile consecutive outputs of one microphone; the input is consumed in
// chunks that never straddle a segment boundary, so each chunk uses one RIR, whose needed slice is
// staged in shared memory with a 1-in-32 padding (conflict-free stride-8 reads).  Every thread keeps 8
// consecutive outputs in registers and a sliding 8-tap window of the RIR, so each input sample costs one
// shared load of the RIR, one broadcast load of the signal and 8 FFMA.
#include "kernels.h"

namespace gpurir {

constexpr int kCvThreads = 256;
constexpr int kCvPer = 8;                        // consecutive outputs per thread
constexpr int kCvTile = kCvThreads * kCvPer;     // 2048 outputs per CTA
constexpr int kCvChunk = 256;                    // input samples per shared-memory chunk
constexpr int kCvSlice = kCvTile + kCvChunk;     // RIR taps needed by one chunk (+1 spare)

__host__ __device__ constexpr int cv_pad(int e) { return e + (e >> 5); }

__global__ void __launch_bounds__(kCvThreads) traj_kernel(const float* __restrict__ sig, long long n_sig,
                                                           const float* __restrict__ rirs, int n_points, int n_mics,
                                                           long long L, float* __restrict__ out) {
  __shared__ float s_sig[kCvChunk];
  __shared__ float s_rir[cv_pad(kCvSlice) + 1];
  const int tid = threadIdx.x;
  const int m = blockIdx.y;
  const long long n_out = n_sig + L - 1;
  const long long t0 = (long long)blockIdx.x * kCvTile;
  const long long seglen = n_sig / n_points;
  float acc[kCvPer];
#pragma unroll
  for (int i = 0; i < kCvPer; i++) acc[i] = 0.f;

  // inputs that reach outputs [t0, t0 + kCvTile): t - L < j <= t
  const long long jlo = t0 - L + 1 > 0 ? t0 - L + 1 : 0;
  const long long jhi = t0 + kCvTile < n_sig ? t0 + kCvTile : n_sig;
  for (long long jc = jlo; jc < jhi;) {
    long long p = jc / seglen;
    if (p > n_points - 1) p = n_points - 1;
    long long jend = jc + kCvChunk;
    if (jend > jhi) jend = jhi;
    if (p < n_points - 1 && jend > (p + 1) * seglen) jend = (p + 1) * seglen;  // one RIR per chunk
    const int n = (int)(jend - jc);
    // stage the chunk's signal and the RIR slice tau in [t0 - jend + 1, t0 + kCvTile - 1 - jc]
    const float* h = rirs + ((long long)p * n_mics + m) * L;
    const long long tmin = t0 - jend + 1;
    const int nslice = kCvTile + n - 1;
    __syncthreads();  // previous chunk consumed
    for (int i = tid; i < n; i += kCvThreads) s_sig[i] = sig[jc + i];
    for (int e = tid; e < nslice; e += kCvThreads) {
      const long long tau = tmin + e;
      s_rir[cv_pad(e)] = (tau >= 0 && tau < L) ? h[tau] : 0.f;
    }
    __syncthreads();
    // thread outputs t_i = t0 + 8 tid + i; for d = jend - 1 - j the tap index is e = 8 tid + i + d
    float w[kCvPer];
#pragma unroll
    for (int i = 0; i < kCvPer; i++) w[i] = s_rir[cv_pad(kCvPer * tid + i)];
    int d = 0;
    for (; d + kCvPer <= n; d += kCvPer) {
#pragma unroll
      for (int u = 0; u < kCvPer; u++) {  // window rotation is register renaming after unrolling
        const float sv = s_sig[n - 1 - (d + u)];
#pragma unroll
        for (int i = 0; i < kCvPer; i++) acc[i] = fmaf(sv, w[(i + u) % kCvPer], acc[i]);
        w[u] = s_rir[cv_pad(kCvPer * tid + d + u + kCvPer)];
      }
    }
    for (; d < n; d++) {
      const float sv = s_sig[n - 1 - d];
#pragma unroll
      for (int i = 0; i < kCvPer; i++) acc[i] = fmaf(sv, s_rir[cv_pad(kCvPer * tid + i + d)], acc[i]);
    }
    jc = jend;
  }
  float* o = out + (long long)m * n_out;
#pragma unroll
  for (int i = 0; i < kCvPer; i++) {
    const long long t = t0 + kCvPer * tid + i;
    if (t < n_out) o[t] = acc[i];
  }
}

cudaError_t launch_traj(const float* sig, long long n_sig, const float* rirs, int n_points, int n_mics, long long L,
                        float* out, cudaStream_t stream) {
  const long long n_out = n_sig + L - 1;
  dim3 grid((unsigned)((n_out + kCvTile - 1) / kCvTile), (unsigned)n_mics);
  traj_kernel<<<grid, kCvThreads, 0, stream>>>(sig, n_sig, rirs, n_points, n_mics, L, out);
  return cudaGetLastError();
}

}  // namespace gpurir

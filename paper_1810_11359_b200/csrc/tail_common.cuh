// tail_common.cuh — the diffuse tail's per-RIR arithmetic (hot-path rows a6, a7 of SURVEY.md §8(a)), shared
// by tail_kernel (one warp per RIR chunk) and the polyphase kernel's fused tail (the CTA that finishes a
// RIR's last ISM tile), so that both produce the same RIRs bit for bit.
//   P(t) = A_env exp(-kappa t), kappa = 6 ln 10 / T60 (Eq. 8, reading C14), T60 from Sabine (Eq. 7);
//   A_env = mean(h^2) / mean(exp(-kappa k/fs)) over the last 10 ms of ISM before Tdiff, clipped at the
//   direct-path sample (reading C15);
//   h[k] = sqrt(P(k/fs)) * (sqrt(3)/pi) ln(u / (1 - u)),  nISM <= k < nS  (logistic noise),
//   u from the stateless Philox4x32-10 stream (seed, global RIR index, k) (reading C16).
#pragma once
#include "device_common.cuh"

namespace gpurir {

__device__ __forceinline__ float tail_lg2(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float tail_ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Envelope of one RIR by one full warp (every lane returns the same values): h(k) returns ISM sample k.
// env0 = sqrt(A_env exp(-kappa nISM / fs)) (sqrt(3)/pi) ln 2, alpha = -kappa / (2 ln 2 fs), rho = 2^alpha.
template <class HF>
__device__ __forceinline__ void tail_envelope(HF h, int nISM, int win, double x_dp, float kappa_fs, int lane,
                                              float& env0, float& alpha, float& rho) {
  int w0 = nISM - win;
  const int wdp = (int)ceil(x_dp);
  if (wdp > w0) w0 = wdp;
  if (w0 < 0) w0 = 0;
  double sh = 0.0, se = 0.0;
  const float kl2 = -kappa_fs * 1.4426950408889634f;  // exp(-kappa k / fs) = 2^(kl2 k)
  for (int k = w0 + lane; k < nISM; k += 32) {
    const double v = (double)h(k);
    sh += v * v;
    se += (double)tail_ex2(kl2 * (float)(k - w0));  // relative to w0; the common factor is restored below
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {  // fixed butterfly, then lane 0's sums for everyone
    sh += __shfl_xor_sync(0xffffffffu, sh, o);
    se += __shfl_xor_sync(0xffffffffu, se, o);
  }
  sh = __shfl_sync(0xffffffffu, sh, 0);
  se = __shfl_sync(0xffffffffu, se, 0);
  se *= exp(-(double)kappa_fs * (double)w0);
  const double Aenv = (w0 < nISM && se > 0.0) ? sh / se : 0.0;
  // sqrt(P(k)) * sqrt(3)/pi * ln 2 = env0 * 2^(alpha (k - nISM)), alpha = -kappa_fs / (2 ln 2)
  env0 = (float)(sqrt(Aenv * exp(-(double)kappa_fs * nISM)) * 0.5513288954217920495 * 0.69314718055994530942);
  alpha = -kappa_fs * 0.72134752044448170368f;
  rho = tail_ex2(alpha);  // envelope ratio between consecutive samples
}

// One Philox block q (samples 4q .. 4q + 3) of one RIR's tail, written where nISM <= k < nS into row.
__device__ __forceinline__ void tail_quad(long long q, int nISM, int nS, float env0, float alpha, float rho,
                                          const PhiloxKey& key, unsigned long long rglob, float* row,
                                          bool aligned) {
  const uint4 ctr = make_uint4((uint32_t)q, (uint32_t)((unsigned long long)q >> 32), (uint32_t)rglob,
                               (uint32_t)(rglob >> 32));
  const uint4 w = philox4x32_10(ctr, key);
  const long long k0 = q * 4;
  float e = env0 * tail_ex2(alpha * (float)(k0 - nISM));
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
  float vals[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    // u = (2 (w >> 9) + 1) 2^-24 built exactly without an int->float conversion:
    // f = 1 + (w >> 9) 2^-23 in [1, 2), u = f - (1 - 2^-24); 1 - u is an odd multiple of 2^-24 below 1,
    // so it is exact in fp32 too
    const float f = __uint_as_float(0x3F800000u | (ws[j] >> 9));
    const float u = f - 0.99999994039535522461f;
    const float omu = 1.f - u;
    vals[j] = e * (tail_lg2(u) - tail_lg2(omu));  // sqrt(P) (sqrt3/pi) ln(u/(1-u))
    e *= rho;
  }
  float* o = row + k0;
  if (aligned && k0 >= nISM && k0 + 3 < nS) {
    *reinterpret_cast<float4*>(o) = make_float4(vals[0], vals[1], vals[2], vals[3]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const long long k = k0 + j;
      if (k >= nISM && k < nS) o[j] = vals[j];
    }
  }
}

}  // namespace gpurir

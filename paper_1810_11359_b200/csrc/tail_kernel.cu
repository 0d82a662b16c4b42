// tail_kernel.cu — envelope prediction + diffuse tail (hot-path rows a6, a7 of
// SURVEY.md §8(a); envPred + cuRAND + diffRev of Table 2).
//
// Per RIR (§2.2.3):
//   P(t) = A_env exp(-kappa t), kappa = 6 ln 10 / T60 (Eq. 8, reading C14), T60 from Sabine (Eq. 7);
//   A_env = mean(h^2) / mean(exp(-kappa k/fs)) over the last 10 ms of ISM before Tdiff, clipped at
//   the direct-path sample (reading C15);
//   h[k] = sqrt(P(k/fs)) * (sqrt(3)/pi) ln(u / (1 - u)),  nISM <= k < nS  (logistic noise),
//   u from the stateless Philox4x32-10 stream (seed, global RIR index, k) (reading C16).
// One warp per (RIR, chunk of chunk_quads Philox blocks).  Each warp re-reduces the
// envelope window (<= 480 floats, L2 hits, fp64 sums, fixed butterfly) so the
// tail needs no separate launch and no scratch; the RNG has no seeding kernel
// and no noise buffer in HBM.  Output writes (4 B / sample, float4 stores) are
// the only HBM traffic.
#include "device_common.cuh"
#include "kernels.h"

namespace gpurir {

__device__ __forceinline__ float lg2_approx(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float ex2_fast(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// One warp per (RIR, chunk): the envelope window is reduced with warp shuffles
// only (no block barriers), so the short prologue of one warp overlaps the streaming stores of others.
__global__ void __launch_bounds__(kTailThreads) tail_kernel(TailArgs A, long long n_items) {
  const int lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * (kTailThreads / 32) + (threadIdx.x >> 5);
  if (item >= n_items) return;

  int rir, chunk, nISM, nS;
  long long row;
  float kappa_fs;
  unsigned long long rglob;
  const float* ps;
  const float* pr;
  if (A.jobs) {
    int2 jc = A.chunks[item];
    rir = jc.x; chunk = jc.y;
    const BatchJob& J = A.jobs[rir];
    nISM = J.nISM; nS = J.nS; row = J.out_offset; kappa_fs = J.kappa_fs; rglob = J.rir_global;
    ps = J.src; pr = J.rcv;
  } else {
    rir = (int)(item / A.chunks_per_rir);
    chunk = (int)(item % A.chunks_per_rir);
    nISM = A.nISM; nS = A.nS; row = (long long)rir * A.row_stride; kappa_fs = A.kappa_fs;
    rglob = A.rir_base + (unsigned long long)rir;
    ps = A.pos_src + 3 * (rir / A.M_rcv);
    pr = A.pos_rcv + 3 * (rir % A.M_rcv);
  }
  const float* h = A.out + row;

  // ---- envelope prediction (envPred; C15) -------------------------------
  const double ddx = (double)ps[0] - pr[0], ddy = (double)ps[1] - pr[1], ddz = (double)ps[2] - pr[2];
  const double x_dp = sqrt(ddx * ddx + ddy * ddy + ddz * ddz) * A.fs_over_c;  // direct-path delay (samples)
  int w0 = nISM - A.win;
  const int wdp = (int)ceil(x_dp);
  if (wdp > w0) w0 = wdp;
  if (w0 < 0) w0 = 0;
  double sh = 0.0, se = 0.0;
  const float kl2 = -kappa_fs * 1.4426950408889634f;  // exp(-kappa k / fs) = 2^(kl2 k)
  for (int k = w0 + lane; k < nISM; k += 32) {
    const double v = (double)h[k];
    sh += v * v;
    se += (double)ex2_fast(kl2 * (float)(k - w0));    // relative to w0; the common factor is restored below
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
  const float env0 = (float)(sqrt(Aenv * exp(-(double)kappa_fs * nISM)) * 0.5513288954217920495 *
                             0.69314718055994530942);
  const float alpha = -kappa_fs * 0.72134752044448170368f;
  const float rho = ex2_fast(alpha);  // envelope ratio between consecutive samples

  // ---- tail samples: Philox blocks of 4 samples ----------------------------------
  const long long q0 = (long long)(nISM >> 2);
  const long long qend = (long long)((nS + 3) >> 2);
  const PhiloxKey key = philox_key(make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32)));
  const bool aligned = ((row & 3) == 0);
  const long long qbeg = q0 + (long long)chunk * A.chunk_quads;
  const long long qlim = min(qend, qbeg + (long long)A.chunk_quads);
#pragma unroll 2
  for (long long q = qbeg + lane; q < qlim; q += 32) {
    const uint4 ctr = make_uint4((uint32_t)q, (uint32_t)((unsigned long long)q >> 32), (uint32_t)rglob,
                                 (uint32_t)(rglob >> 32));
    const uint4 w = philox4x32_10(ctr, key);
    const long long k0 = q * 4;
    float e = env0 * ex2_fast(alpha * (float)(k0 - nISM));
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
      vals[j] = e * (lg2_approx(u) - lg2_approx(omu));  // sqrt(P) (sqrt3/pi) ln(u/(1-u))
      e *= rho;
    }
    float* o = A.out + row + k0;
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
}

cudaError_t launch_tail(const TailArgs& A, long long n_items, cudaStream_t stream) {
  if (n_items <= 0) return cudaSuccess;
  const long long per = kTailThreads / 32;
  tail_kernel<<<(unsigned)((n_items + per - 1) / per), kTailThreads, 0, stream>>>(A, n_items);
  return cudaGetLastError();
}

}  // namespace gpurir

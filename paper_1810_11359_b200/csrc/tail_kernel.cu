// tail_kernel.cu — envelope prediction + diffuse tail (hot-path rows a6, a7 of
// SURVEY.md §8(a); envPred + cuRAND + diffRev of Table 2).
//
// Per RIR (§2.2.3):
//   P(t) = A_env exp(-kappa t), kappa = 6 ln 10 / T60 (Eq. 8, reading C14), T60 from Sabine (Eq. 7);
//   A_env = mean(h^2) / mean(exp(-kappa k/fs)) over the last 10 ms of ISM before Tdiff, clipped at
//   the direct-path sample (reading C15);
//   h[k] = sqrt(P(k/fs)) * (sqrt(3)/pi) ln(u / (1 - u)),  nISM <= k < nS  (logistic noise),
//   u from the stateless Philox4x32-10 stream (seed, global RIR index, k) (reading C16).
// The envelope window is re-reduced by every CTA of the RIR (<= 480 samples from L2)
// so the tail needs no separate launch and no scratch; the RNG has no seeding
// kernel and no noise buffer in HBM.  Output writes are the only HBM traffic.
#include "device_common.cuh"
#include "kernels.h"

namespace gpurir {

__global__ void __launch_bounds__(kTailThreads) tail_kernel(TailArgs A) {
  __shared__ double red_h[kTailThreads / 32], red_e[kTailThreads / 32];
  __shared__ float s_env0, s_alpha;

  int rir, chunk, nISM, nS;
  long long row;
  float kappa_fs;
  unsigned long long rglob;
  float sx, sy, sz, rx, ry, rz;
  if (A.jobs) {
    int2 jc = A.chunks[blockIdx.x];
    rir = jc.x; chunk = jc.y;
    const BatchJob& J = A.jobs[rir];
    nISM = J.nISM; nS = J.nS; row = J.out_offset; kappa_fs = J.kappa_fs; rglob = J.rir_global;
    sx = J.src[0]; sy = J.src[1]; sz = J.src[2]; rx = J.rcv[0]; ry = J.rcv[1]; rz = J.rcv[2];
  } else {
    rir = blockIdx.x / A.chunks_per_rir;
    chunk = blockIdx.x % A.chunks_per_rir;
    nISM = A.nISM; nS = A.nS; row = (long long)rir * A.row_stride; kappa_fs = A.kappa_fs;
    rglob = A.rir_base + (unsigned long long)rir;
    int ms = rir / A.M_rcv, mr = rir % A.M_rcv;
    sx = A.pos_src[3 * ms]; sy = A.pos_src[3 * ms + 1]; sz = A.pos_src[3 * ms + 2];
    rx = A.pos_rcv[3 * mr]; ry = A.pos_rcv[3 * mr + 1]; rz = A.pos_rcv[3 * mr + 2];
  }
  const float* h = A.out + row;
  const int tid = threadIdx.x;

  // ---- envelope prediction (envPred; C15) -------------------------------
  double ddx = (double)sx - rx, ddy = (double)sy - ry, ddz = (double)sz - rz;
  double x_dp = sqrt(ddx * ddx + ddy * ddy + ddz * ddz) * A.fs_over_c;
  int w0 = nISM - A.win;
  int wdp = (int)ceil(x_dp);
  if (wdp > w0) w0 = wdp;
  if (w0 < 0) w0 = 0;
  double sh = 0.0, se = 0.0;
  for (int k = w0 + tid; k < nISM; k += kTailThreads) {
    double v = (double)h[k];
    sh += v * v;
    se += exp(-(double)kappa_fs * (double)k);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sh += __shfl_xor_sync(0xffffffffu, sh, o);
    se += __shfl_xor_sync(0xffffffffu, se, o);
  }
  if ((tid & 31) == 0) { red_h[tid >> 5] = sh; red_e[tid >> 5] = se; }
  __syncthreads();
  if (tid == 0) {
    double th = 0.0, te = 0.0;
    for (int w = 0; w < kTailThreads / 32; w++) { th += red_h[w]; te += red_e[w]; }
    double Aenv = (w0 < nISM && te > 0.0) ? th / te : 0.0;
    // sqrt(P(k)) = sqrt(Aenv exp(-kappa nISM/fs)) * 2^(-kappa_fs (k - nISM) / (2 ln 2))
    s_env0 = (float)(sqrt(Aenv * exp(-(double)kappa_fs * nISM)) * 0.5513288954217920495);  // * sqrt(3)/pi
    s_alpha = -kappa_fs * 0.72134752044448170368f;  // -kappa_fs / (2 ln 2)
  }
  __syncthreads();
  const float env0 = s_env0, alpha = s_alpha;

  // ---- tail samples: 2 Philox blocks (8 samples) per thread ---------------------
  const long long q0 = (long long)(nISM >> 2);
  const long long qend = (long long)((nS + 3) >> 2);
  const uint2 key = make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32));
  const float ln2 = 0.69314718055994530942f;
#pragma unroll
  for (int half = 0; half < 2; half++) {
    long long q = q0 + (long long)chunk * (kTailChunk / 4) + half * kTailThreads + tid;
    if (q >= qend) break;
    uint4 ctr = make_uint4((uint32_t)q, (uint32_t)((unsigned long long)q >> 32), (uint32_t)rglob,
                           (uint32_t)(rglob >> 32));
    uint4 w = philox4x32_10(ctr, key);
    uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    float vals[4];
    long long k0 = q * 4;
#pragma unroll
    for (int j = 0; j < 4; j++) {
      float a = (float)(2u * (ws[j] >> 9) + 1u);  // u = a 2^-24, 1 - u = b 2^-24 (exact)
      float b = 16777216.f - a;
      float lg = (__log2f(a) - __log2f(b)) * ln2;  // ln(u / (1 - u))
      float env = env0 * exp2f(alpha * (float)(k0 + j - nISM));
      vals[j] = env * lg;
    }
    float* o = A.out + row + k0;
    bool full = (k0 >= nISM) && (k0 + 3 < nS);
    if (full && (((row + k0) & 3) == 0)) {
      *reinterpret_cast<float4*>(o) = make_float4(vals[0], vals[1], vals[2], vals[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        long long k = k0 + j;
        if (k >= nISM && k < nS) o[j] = vals[j];
      }
    }
  }
}

cudaError_t launch_tail(const TailArgs& A, long long nblocks, cudaStream_t stream) {
  if (nblocks <= 0) return cudaSuccess;
  tail_kernel<<<(unsigned)nblocks, kTailThreads, 0, stream>>>(A);
  return cudaGetLastError();
}

}  // namespace gpurir

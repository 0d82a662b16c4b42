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
#include "tail_common.cuh"
#include "kernels.h"

namespace gpurir {

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
  float env0, alpha, rho;
  tail_envelope([&](int k) { return h[k]; }, nISM, A.win, x_dp, kappa_fs, lane, env0, alpha, rho);

  // ---- tail samples: Philox blocks of 4 samples ----------------------------------
  const long long q0 = (long long)(nISM >> 2);
  const long long qend = (long long)((nS + 3) >> 2);
  const PhiloxKey key = philox_key(make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32)));
  const bool aligned = (reinterpret_cast<uintptr_t>(A.out + row) & 15) == 0;  // float4 stores: 16-B row start
  const long long qbeg = q0 + (long long)chunk * A.chunk_quads;
  const long long qlim = min(qend, qbeg + (long long)A.chunk_quads);
#pragma unroll 2
  for (long long q = qbeg + lane; q < qlim; q += 32)
    tail_quad(q, nISM, nS, env0, alpha, rho, key, rglob, A.out + row, aligned);
}

cudaError_t launch_tail(const TailArgs& A, long long n_items, cudaStream_t stream) {
  if (n_items <= 0) return cudaSuccess;
  const long long per = kTailThreads / 32;
  tail_kernel<<<(unsigned)((n_items + per - 1) / per), kTailThreads, 0, stream>>>(A, n_items);
  return cudaGetLastError();
}

}  // namespace gpurir

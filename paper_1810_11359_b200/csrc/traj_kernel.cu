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
// staged in shared memory (cp.async, double-buffered so the next chunk's loads overlap this chunk's
// FMAs) with a 1-in-32 padding (conflict-free stride-16 reads).  Every thread keeps 16
// consecutive outputs in registers (paired for FFMA2) and a sliding 16-tap window of the RIR, so each input
// sample costs one shared load of the RIR, a quarter of a float4 broadcast load of the signal and 8 FFMA2.
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace gpurir {

constexpr int kCvThreads = 128;
constexpr int kCvPer = 16;                       // consecutive outputs per thread
constexpr int kCvTile = kCvThreads * kCvPer;     // 2048 outputs per CTA
constexpr int kCvChunk = 512;                    // input samples per shared-memory chunk
constexpr int kCvSlice = kCvTile + kCvChunk;     // RIR taps needed by one chunk (+1 spare)

__host__ __device__ constexpr int cv_pad(int e) { return e + (e >> 5); }

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

struct CvChunk {
  long long jc, jend, p;
};

// The next chunk at jc: at most kCvChunk inputs, never past jhi, never across a segment boundary.
__device__ __forceinline__ CvChunk cv_chunk(long long jc, long long jhi, long long seglen, int n_points) {
  CvChunk c;
  c.jc = jc;
  c.p = jc / seglen;
  if (c.p > n_points - 1) c.p = n_points - 1;
  c.jend = jc + kCvChunk;
  if (c.jend > jhi) c.jend = jhi;
  if (c.p < n_points - 1 && c.jend > (c.p + 1) * seglen) c.jend = (c.p + 1) * seglen;  // one RIR per chunk
  return c;
}

__global__ void __launch_bounds__(kCvThreads) traj_kernel(const float* __restrict__ sig, long long n_sig,
                                                           const float* __restrict__ rirs, int n_points, int n_mics,
                                                           long long L, float* __restrict__ out) {
  __shared__ __align__(16) float s_sig[2][kCvChunk];  // each chunk's signal, time-reversed (double buffer)
  __shared__ float s_rir[2][cv_pad(kCvSlice) + 1];
  const int tid = threadIdx.x;
  const int m = blockIdx.y;
  const long long n_out = n_sig + L - 1;
  const long long seglen = n_sig / n_points;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int crank = (int)cluster.block_rank();
  const long long t0 = (long long)(blockIdx.x / cs) * kCvTile;
  float2 acc2[kCvPer / 2];  // outputs (i, i + 8) of this thread's 16
#pragma unroll
  for (int i = 0; i < kCvPer / 2; i++) acc2[i] = make_float2(0.f, 0.f);

  // stage chunk c: its signal and the RIR slice tau in [t0 - jend + 1, t0 + kCvTile - 1 - jc]
  auto stage = [&](const CvChunk& c, int buf) {
    const float* h = rirs + ((long long)c.p * n_mics + m) * L;
    const long long tmin = t0 - c.jend + 1;
    const int n = (int)(c.jend - c.jc);
    const int nslice = kCvTile + n - 1;
    const float* sg = sig + (c.jend - 1);
    for (int i = tid; i < n; i += kCvThreads) cp_async4(&s_sig[buf][i], sg - i, true);
    // slice element e holds tau = tmin + e; valid taps are e in [elo, ehi), zero-filled elsewhere
    const int elo = tmin < 0 ? (int)(-tmin) : 0;
    const long long eh = L - tmin;
    const int ehi = eh < nslice ? (int)eh : nslice;
    const float* hb = h + tmin;  // only dereferenced for valid e
    float* dst = &s_rir[buf][cv_pad(tid)];  // cv_pad(tid + 128 k) = cv_pad(tid) + 132 k
    for (int e = tid; e < nslice; e += kCvThreads, dst += kCvThreads + kCvThreads / 32) {
      const bool ok = e >= elo && e < ehi;
      cp_async4(dst, ok ? hb + e : h, ok);
    }
    cp_async_commit();
  };

  // inputs that reach outputs [t0, t0 + kCvTile): t - L < j <= t, split into cs equal pieces (one per CTA
  // of the cluster, multiples of kCvPer) so long RIRs do not serialise a tile on one CTA
  const long long tlo = t0 - L + 1 > 0 ? t0 - L + 1 : 0;
  const long long thi = t0 + kCvTile < n_sig ? t0 + kCvTile : n_sig;
  const long long piece = ((thi - tlo + cs - 1) / cs + kCvPer - 1) / kCvPer * kCvPer;
  const long long jlo = tlo + crank * piece;
  const long long jhi = jlo + piece < thi ? jlo + piece : thi;
  if (jlo < jhi) {
    CvChunk cur = cv_chunk(jlo, jhi, seglen, n_points);
    stage(cur, 0);
    for (int buf = 0;; buf ^= 1) {
      const bool more = cur.jend < jhi;
      CvChunk nxt;
      if (more) {
        nxt = cv_chunk(cur.jend, jhi, seglen, n_points);
        stage(nxt, buf ^ 1);  // overlaps this chunk's FMAs
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      // thread outputs t_i = t0 + kCvPer tid + i; input j = jend - 1 - d meets tap e = kCvPer tid + i + d
      const float* sr = s_rir[buf];
      const float* ss = s_sig[buf];
      const int n = (int)(cur.jend - cur.jc);
      const int e0 = kCvPer * tid;
      // for a base b that is a multiple of 16 and u < 16, cv_pad(b + u) = cv_pad(b) + u: one address per step.
      // Outputs pair up as (i, i + 8) in float2 accumulators so that one FFMA2 serves two outputs; the
      // 16-tap sliding window is kept twice as register pairs, W2[k] = (w[k], w[k + 8]) and its swap
      // W2s[k] = (w[k + 8], w[k]): the taps (w[a], w[a + 8 mod 16]) a pair needs are W2[a] or W2s[a - 8].
      float2 W2[8], W2s[8];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const float lo = sr[cv_pad(e0) + k], hi = sr[cv_pad(e0) + k + 8];
        W2[k] = make_float2(lo, hi);
        W2s[k] = make_float2(hi, lo);
      }
      int d = 0;
      for (; d + kCvPer <= n; d += kCvPer) {
        const float* rp = sr + cv_pad(e0 + d + kCvPer);
#pragma unroll
        for (int u4 = 0; u4 < kCvPer; u4 += 4) {
          const float4 sv4 = *reinterpret_cast<const float4*>(&ss[d + u4]);  // broadcast
          const float sv[4] = {sv4.x, sv4.y, sv4.z, sv4.w};
#pragma unroll
          for (int uu = 0; uu < 4; uu++) {
            const int u = u4 + uu;  // all indices below are compile-time after unrolling
            const float2 s2 = make_float2(sv[uu], sv[uu]);
#pragma unroll
            for (int i = 0; i < 8; i++) {
              const int a = (i + u) & 15;
              acc2[i] = __ffma2_rn(s2, a < 8 ? W2[a] : W2s[a - 8], acc2[i]);
            }
            const float v = rp[u];  // the tap entering window slot u
            if (u < 8) { W2[u].x = v; W2s[u].y = v; } else { W2[u - 8].y = v; W2s[u - 8].x = v; }
          }
        }
      }
      for (; d < n; d++) {
        const float sv = ss[d];
#pragma unroll
        for (int i = 0; i < 8; i++)
          acc2[i] = __ffma2_rn(make_float2(sv, sv), make_float2(sr[cv_pad(e0 + i + d)], sr[cv_pad(e0 + i + 8 + d)]),
                               acc2[i]);
      }
      __syncthreads();  // buffer consumed before the next iteration stages into it
      if (!more) break;
      cur = nxt;
    }
  }
  float acc[kCvPer];
#pragma unroll
  for (int i = 0; i < kCvPer / 2; i++) { acc[i] = acc2[i].x; acc[i + 8] = acc2[i].y; }
  float* o = out + (long long)m * n_out;
  if (cs == 1) {
#pragma unroll
    for (int i = 0; i < kCvPer; i++) {
      const long long t = t0 + kCvPer * tid + i;
      if (t < n_out) o[t] = acc[i];
    }
    return;
  }
  // cluster reduction over DSMEM in fixed rank order (deterministic): partials to smem, then rank r sums
  // outputs [r kCvTile / cs, (r + 1) kCvTile / cs) over ranks 0..cs-1 and writes them coalesced
  float* red = &s_rir[0][0];
#pragma unroll
  for (int i = 0; i < kCvPer; i++) red[cv_pad(kCvPer * tid + i)] = acc[i];
  cluster.sync();
  const int span = kCvTile / cs;
  for (int k = tid; k < span; k += kCvThreads) {
    const int e = crank * span + k;
    float v = 0.f;
    for (int q = 0; q < cs; q++) v += cluster.map_shared_rank(red, q)[cv_pad(e)];
    const long long t = t0 + e;
    if (t < n_out) o[t] = v;
  }
  cluster.sync();  // keep this CTA's partials alive until every rank has read them
}

cudaError_t launch_traj(const float* sig, long long n_sig, const float* rirs, int n_points, int n_mics, long long L,
                        float* out, cudaStream_t stream) {
  const long long n_out = n_sig + L - 1;
  const long long n_tiles = (n_out + kCvTile - 1) / kCvTile;
  // a tile reads up to kCvTile + L - 1 inputs; split them over a cluster of cs CTAs until either every tile
  // has at most ~2 chunks per CTA or cs reaches the portable cluster limit
  const long long most = kCvTile + L - 1 < n_sig ? kCvTile + L - 1 : n_sig;
  int cs = 1;
  while (cs < 8 && most > (long long)cs * 2 * kCvChunk) cs *= 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_tiles * cs), (unsigned)n_mics, 1);
  cfg.blockDim = dim3(kCvThreads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, traj_kernel, sig, n_sig, rirs, n_points, n_mics, L, out);
}

}  // namespace gpurir

// ism_poly_kernel.cu — polyphase ISM accumulation, "bin then filter" (mode GPURIR_POLY; hot-path rows
// a1-a3 of SURVEY.md §8(a), reading R11 of DESIGN.md).
//
// Eq. 5 with the windowed sinc of Eq. 6 sums A_n delta'(k - x_n) over every image n and
// sample k.  Writing x_n = j_n + phi_n (j_n = floor(x_n)) and expanding delta' on each integer tap
// m = k - j_n in Chebyshev polynomials of the fractional delay,
//     delta'(m - phi) = sum_d P_d[m] T_d(2 phi - 1),   d = 0..7   (max error 4.3e-7, host fit),
// the RIR becomes a fixed 8-channel FIR filter applied to per-sample image aggregates:
//     h[k] = sum_m sum_d P_d[m] G_d[k - m],   G_d[j] = sum_{n: j_n = j} A_n T_d(2 phi_n - 1).
// Persistent CTAs (THREADS = 256 x 4 per SM from 7 items per SM, 512 x 2 below, 1024 x 1 for calls of at most
// one item per SM; calls of <= 2 items per SM split their heavy tiles' output ranges over the free CTA slots)
// take (RIR, 1024-sample tile) work items from a global counter; per item the CTA
//   1. enumerates the tile's shell of images column by column (as ism_ws_kernel; nonempty columns
//      compacted by the candidate scan) and adds each image's 8 channel values into G in shared memory —
//      as fixed point with integer reductions (one int32 word per channel, or two for tiles dense enough to
//      need them; the scale is per tile), so the sums are exact and independent of the order the images
//      arrive in (deterministic, shard-invariant); the fraction of the delay comes from the exact floor of
//      the fp32 estimate plus its fp64 correction;
//   2. converts G to fp32 in place, rotates each position's 8 values by Q (reading R13: G' = Q G, per parity)
//      and runs the FIR: rotated channels 0..3 over all 2H taps, 4..7 over an 8-tap window around the image
//      (288 instead of 512 MACs per output at 16 kHz), 4 partials x 8 consecutive outputs per thread item with a
//      sliding register window, partial sums meeting in shared memory; the tile is written once, coalesced.
// Small calls (<= 32 items) run cluster items instead: a tile's columns split over a thread-block cluster whose
// ranks' integer planes meet through L2 (same bits as the persistent CTAs).
// The kernel is bound by shared-memory wavefronts (80 % of peak: the random-position reductions and the
// FIR's loads), so the loops keep their constants in registers rather than re-reading them from shared
// memory.
// Work per output sample no longer grows with the image density (690 in-window taps per sample at config
// 3 (i)): the filter costs 4 x 2H + 4 x 8 MACs, the aggregation 8 channel updates per image.
#include <cooperative_groups.h>
#include <algorithm>
#include <mutex>
#include <utility>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "ism_common.cuh"
#include "tail_common.cuh"

namespace cg = cooperative_groups;

namespace gpurir {

// Phase timing of the cluster items (diagnostic build -DGPURIR_PHASE_TIMING, tools/build_variant.sh,
// tools/phase_probe.py): thread 0 of every CTA prints %globaltimer at the phase boundaries of its item
#ifdef GPURIR_PHASE_TIMING
#define PT_MARK(i) do { if (threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); pt_[i] = t_; } } while (0)
#define PT_DUMP() do { if (threadIdx.x == 0) printf("PT %d %d %d %d %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", (int)blockIdx.x, (int)sm.ti.rir, 0, 1, pt_[0], pt_[1], pt_[2], pt_[3], pt_[4], pt_[5], pt_[6], pt_[7], (unsigned long long)sm.ti.te, pts_[0], pts_[1], pts_[2], pts_[3], pts_[4]); } while (0)
// setup sub-steps of thread 0 (SM clock, for differences within the CTA): kernel entry, after the P table load,
// after the item decode, after geom_from; the PT line also prints the clock at the end of the setup
#define PS_MARK(i) do { if (threadIdx.x == 0) pts_[i] = clock64(); } while (0)
#else
#define PT_MARK(i) do {} while (0)
#define PS_MARK(i) do {} while (0)
#define PT_DUMP() do {} while (0)
#endif
// persistent items (the same build): per-phase time summed over the items of CTAs 0..7, printed at their exit
#ifdef GPURIR_PHASE_TIMING
#define PTL_MARK(i) do { if (threadIdx.x == 0) { unsigned long long t_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); ptl_[i] = t_; } } while (0)
#define PTL_ACC() do { if (threadIdx.x == 0) { for (int i_ = 1; i_ < 7; i_++) pta_[i_] += ptl_[i_] - ptl_[i_ - 1]; pta_[0]++; } } while (0)
#define PTL_DUMP() do { if (threadIdx.x == 0 && blockIdx.x < 8) printf("PTL %d items %llu setup %llu bz %llu aggr %llu conv %llu fir %llu end %llu\n", (int)blockIdx.x, pta_[0], pta_[1], pta_[2], pta_[3], pta_[4], pta_[5], pta_[6]); } while (0)
#else
#define PTL_MARK(i) do {} while (0)
#define PTL_ACC() do {} while (0)
#define PTL_DUMP() do {} while (0)
#endif

constexpr int kPolyTC = kPolyTile;      // output samples per work item (the host planner's tile)
constexpr int kPolyD = 8;               // Chebyshev channels T_0..T_7
constexpr int kPolyBz = 1024;           // z-factor table entries
// CTA shape (template parameter THREADS, 512 or 256): 1024 / THREADS CTAs per SM at 64 registers per thread
template <int THREADS> struct PolyCfg {
  static constexpr int kThreads = THREADS;
  static constexpr int kCtasPerSm = THREADS >= 1024 ? 1 : 1024 / THREADS;
  static constexpr int kCols = THREADS;         // lattice columns per enumeration batch
  static constexpr int kGroup = THREADS / 4;    // FIR threads per channel pair
  static constexpr int kPass = 8 * kGroup;      // outputs per FIR pass (8 per thread)
  // FIR items (4 partials x kPolyTC / 8 blocks of 8 outputs) per thread: 2 (256 threads), 1 (512), 1 with half the
  // threads idle (1024: persistent CTAs of calls with at most one item per SM, and cluster items)
  static constexpr int kPasses = THREADS >= 1024 ? 1 : kPolyTC / kPass;
  static_assert(THREADS >= 1024 || kPolyTC % kPass == 0, "FIR passes of 4 channel-pair groups x 8 outputs per thread");
};

// One nonempty lattice column of a batch (32 B, two 16-B loads; lengths in samples, x fs / c).  Its
// candidates are the global indices [start, end) of the batch's candidate list; candidate gi is the image
// n_z = gi + (gi < b ? a1 : a2) (the two n_z runs of the column, see the walk).
struct PolyColRec {
  double rho2;
  float bxy, cdot;
  int a1, a2, b, end;
};
__device__ __forceinline__ PolyColRec load_col(const PolyColRec* c) {
  const int4* p = reinterpret_cast<const int4*>(c);
  const int4 u = p[0], v = p[1];
  PolyColRec r;
  r.rho2 = __hiloint2double(u.y, u.x);
  r.bxy = __int_as_float(u.z);
  r.cdot = __int_as_float(u.w);
  r.a1 = v.x; r.a2 = v.y; r.b = v.z; r.end = v.w;
  return r;
}


struct PolyTile {
  RirGeom g;
  double dlo2, dhi2, invLz, inv_scale;
  double Lzs, offEs, offOs;     // Eq. 1 along z in samples: Delta_z fs / c = n Lz fs / c + off (even / odd n)
  float scalef;      // 2^(bits - e): a power of two, exact in fp32
  float inv_scalef;  // 2^(e - bits), the same as inv_scale
  float scale_lf;    // single word: the last channel's scale 2^(bits - e - J)
  int two_word;
  int e, bits;       // amplitude bound |A| < 2^e (in 1/(fs/c 4 pi) units, see setup); channel resolution bits
  int J;             // the last channel's word counts its deposits in its low J bits (capacity 2^J per position)
  unsigned cnt_mask; // 2^J - 1
  int ovf, redo;     // some position's count reached 2^J / the aggregation is redone at a wider format
  long long row;
  int t0, te, tc, nx0, ny0, NX, ncols, zl, zh, use_bz, next;
  int rir, tail;     // the RIR; this tile ends its ISM part and the call fuses the tail
  int tail_nS;       // fused tail: the RIR's samples, its Philox stream (global RIR index) and decay
  float tail_kappa;
  unsigned long long tail_rglob;
  double x_dp;       // direct-path delay (samples)
  float tenv[3];     // fused tail: env0, alpha, rho of the RIR (tail_envelope)
  float invNX;
  int ot0, ote, npos_i;  // this item's outputs [ot0, ote) and positions (sub-range of the tile; cluster items)
};

// The diffuse tail of RIR T.rir, by the CTA that just wrote its last ISM tile (output partial sums still in
// red): warp 0 reduces the envelope window from shared memory exactly as tail_kernel does from global memory,
// then every thread writes Philox blocks of the tail.  Not inlined: the tail's registers (Philox round keys)
// stay out of the image loop's allocation.
// The diffuse tail of the tile's RIR (tail_common.cuh, bit-identical to tail_kernel): warp 0 reduces the envelope
// window — from the output partial sums still in shared memory (`red`, single-CTA items) or from the samples just
// written to global memory (`hg`, cluster items) — then this CTA writes Philox blocks q0 + tid, + stride, ...
// Not inlined: the tail's registers (Philox round keys) stay out of the image loop's allocation.
__device__ __noinline__ void poly_fused_tail(PolyTile& T, const float* red, const float* hg, int tid, int nthreads,
                                             float* out, int win, unsigned long long seed, int q_first,
                                             int q_stride) {
  const int nISM = T.te, nS = T.tail_nS;
  if (tid < 32) {
    float env0, alpha, rho;
    const int t0 = T.ot0;  // red holds the item's outputs (the last sub-range of a split tile holds the window)
    if (hg)
      tail_envelope([&](int k) { return hg[k]; }, nISM, win, T.x_dp, T.tail_kappa, tid, env0, alpha, rho);
    else
      tail_envelope([&](int k) {
                      const int t = k - t0;
                      return (red[t] + red[kPolyTC + t]) + (red[2 * kPolyTC + t] + red[3 * kPolyTC + t]);
                    },
                    nISM, win, T.x_dp, T.tail_kappa, tid, env0, alpha, rho);
    if (tid == 0) { T.tenv[0] = env0; T.tenv[1] = alpha; T.tenv[2] = rho; }
  }
  __syncthreads();
  const float env0 = T.tenv[0], alpha = T.tenv[1], rho = T.tenv[2];
  const PhiloxKey key = philox_key(make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  float* row = out + T.row;
  const bool aligned = (reinterpret_cast<uintptr_t>(row) & 15) == 0;  // float4 stores need a 16-B row start
  const long long qend = (long long)((nS + 3) >> 2);
  for (long long q = (long long)(nISM >> 2) + q_first + tid; q < qend; q += q_stride)
    tail_quad(q, nISM, nS, env0, alpha, rho, key, T.tail_rglob, row, aligned);
  (void)nthreads;
}

// The fused tail of a cluster item (every rank of the tail tile's cluster calls it): the same samples as
// poly_fused_tail, but each thread first computes its first Philox block's noise (Philox words, the logistic
// transform and the envelope's decay factor; none of it depends on the envelope's level env0) while the cluster
// waits for every rank's outputs; after the envelope only the level multiplies in, in tail_quad's order (same bits).
__device__ __noinline__ void poly_fused_tail_cl(PolyTile& T, const float* hg, int tid, float* out, int win,
                                                unsigned long long seed, int q_first, int q_stride) {
  const int nISM = T.te, nS = T.tail_nS;
  const float alpha = -T.tail_kappa * 0.72134752044448170368f, rho = tail_ex2(alpha);  // as tail_envelope
  const PhiloxKey key = philox_key(make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const long long qend = (long long)((nS + 3) >> 2), q = (long long)(nISM >> 2) + q_first + tid;
  float L[4] = {0.f, 0.f, 0.f, 0.f}, x = 0.f;
  if (q < qend) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)((unsigned long long)q >> 32),
                                             (uint32_t)T.tail_rglob, (uint32_t)(T.tail_rglob >> 32)), key);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const float f = __uint_as_float(0x3F800000u | (ws[j] >> 9));
      const float u = f - 0.99999994039535522461f;
      L[j] = tail_lg2(u) - tail_lg2(1.f - u);
    }
    x = tail_ex2(alpha * (float)(q * 4 - nISM));
  }
  __threadfence();
  cg::this_cluster().sync();  // the tile's samples are in global memory once every rank is here
  if (tid < 32) {
    float env0, a_, r_;
    tail_envelope([&](int k) { return hg[k]; }, nISM, win, T.x_dp, T.tail_kappa, tid, env0, a_, r_);
    if (tid == 0) T.tenv[0] = env0;
  }
  __syncthreads();
  const float env0 = T.tenv[0];
  float* row = out + T.row;
  const bool aligned = (reinterpret_cast<uintptr_t>(row) & 15) == 0;
  if (q < qend) {  // tail_quad's last steps for the precomputed block
    float e = env0 * x, vals[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      vals[j] = e * L[j];
      e *= rho;
    }
    const long long k0 = q * 4;
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
  for (long long qq = q + q_stride; qq < qend; qq += q_stride)
    tail_quad(qq, nISM, nS, env0, alpha, rho, key, T.tail_rglob, row, aligned);
}

template <int THREADS>
struct alignas(16) PolySmem {
  PolyTile ti;
  alignas(16) PolyColRec col[THREADS];  // one lattice column per thread and batch
  int colpre[THREADS];                  // inclusive candidate prefix (= col[].end), for the run search
  float colsdot[THREADS];               // directional source: the column's part of cos(theta_s) (general walk)
  int scan_tmp[THREADS / 32];
  float bz[kPolyBz];
  // persistent single-room items: the next item's queue index and inputs (src, rcv, rcv orientation, src
  // orientation), fetched by thread 0 with cp.async while the current item filters
  long long pf_wi;
  int pf_valid;
  float pf_in[12];
};

// Work entry w of a call with a split plan (IsmArgs::poly_cmap, poly_plan_subs): its item and output sub-range
__device__ __forceinline__ long long poly_decode(const IsmArgs& A, long long w, int& sub, int& nsub) {
  if (A.poly_nitems <= 0) {
    sub = 0;
    nsub = 1;
    return w;
  }
  const int cm = A.poly_cmap[w];
  sub = (cm >> 10) & 3;
  nsub = 1 << (cm >> 12);
  return cm & 0x3FF;
}

// exact q = n / d, r = n % d (0 <= n < 2^53, d >= 1) from a host reciprocal: the fp64 estimate is off by at most one
__device__ __forceinline__ long long poly_divmod(long long n, long long d, double inv_d, long long& r) {
  long long q = (long long)((double)n * inv_d);
  r = n - q * d;
  if (r < 0) { q--; r += d; } else if (r >= d) { q++; r -= d; }
  return q;
}
__device__ __forceinline__ void poly_cp4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

template <int kPolyThreads>
__device__ __forceinline__ int poly_block_scan(int v, int* tmp) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = warp_incl_scan(v, lane);
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < kPolyThreads / 32 ? tmp[lane] : 0;
    t = warp_incl_scan(t, lane);
    if (lane < kPolyThreads / 32) tmp[lane] = t;
  }
  __syncthreads();
  return x + (w > 0 ? tmp[w - 1] : 0);
}

// z-axis factor of beta_n (C2)
__device__ __forceinline__ float poly_z_factor(int nz, const RirGeom& g) {
  uint32_t sgn = 0;
  bool zero = false;
  float lz = axis_beta(nz, 2, g, sgn, zero);
  float v = zero ? 0.f : ex2_approx(lz);
  return sgn ? -v : v;
}

// The same for a single-room call straight from the call's arguments (no RirGeom needed: the z factor reads
// only the z walls' log2 |beta|, signs and zero flags)
__device__ __forceinline__ float poly_z_factor_args(int nz, const IsmArgs& A) {
  RirGeom g;
  g.lb[4] = A.lb[4];
  g.lb[5] = A.lb[5];
  g.neg = A.neg;
  g.zero = A.zero;
  return poly_z_factor(nz, g);
}

// One image's 8 channel values A T_d(y), d = 0..7, added to G[.][p] as integers v = round(A T_d 2^s).  The
// tile's scale bounds |A| by its closest possible image, so |v| <= 2^bits; sums of integers commute, so G does
// not depend on the order in which images arrive (deterministic, shard-invariant).
// Overflow guard (exact, no assumption on how many images share a sample position): the last channel's word
// also COUNTS its deposits, in its low J bits — the channel value goes in shifted left by J (its resolution
// is 2^-J of the others'; its coefficients are <= 8.5e-6, R11) plus 1 — and every deposit reads the word's
// old value.  The deposit that takes a position's count to 2^J sees the count field all ones, so `acc`
// (min over this thread's deposits of ~old & mask) reaches 0 exactly when some position holds 2^J images;
// below that, sum |v| <= (2^J - 1) 2^bits < 2^31 on every channel and no partial sum can wrap.  The tile is
// then redone in a wider format (ism_poly_kernel, after the aggregation).
//   single word (bits <= 22, J = 31 - bits): fp32 arithmetic — T_d by the recurrence in fp32 (|error| ~ 1e-7
//     d), round(A T_d 2^s) from the low mantissa bits of A 2^s T_d + 1.5 2^23 (exact for |v| < 2^22);
//   two words (bits = 28): v = a 2^14 + b, b in [0, 2^14), into two int32 planes (2^17 terms of headroom); the
//     last channel puts round(v 2^-14) in its coarse plane and counts in its fine plane (J = 17).
template <bool kCountFirst>
__device__ __forceinline__ void poly_add(int* Ga, int* Gb, int W, int p, float y, float amp, float scale,
                                         float scale_l, int J, unsigned mask, bool two_word, unsigned& acc) {
  constexpr int kLast = kPolyChannels - 1;
  if (!two_word) {
    // the deposits are the raw bit patterns 0x4B400000 + v of A 2^s T_d + 1.5 2^23: the sums carry count x
    // 0x4B400000 (mod 2^32), removed at the conversion with the exact count of the last channel's low bits
    const float as = amp * scale, y2 = 2.f * y, magic = 12582912.f;  // power-of-two scales: exact
    if constexpr (kCountFirst && kPolyChannels == 8) {  // the counting deposit first: its returned word's latency
                                                          // hides under the other seven (persistent CTAs; see below)
                                         // other seven (+0.2 %, A/B 3 rounds; the same integer sums)
      float Tc[8];
      Tc[0] = 1.f; Tc[1] = y;
#pragma unroll
      for (int d = 2; d < 8; d++) Tc[d] = fmaf(y2, Tc[d - 1], -Tc[d - 2]);
      const unsigned raw = __float_as_uint(fmaf(amp * scale_l, Tc[7], magic));
      const unsigned old = atomicAdd(reinterpret_cast<unsigned*>(&Ga[7 * W + p]), raw * (1u << J) + 1u);
#pragma unroll
      for (int d = 0; d < 7; d++) atomicAdd(&Ga[d * W + p], __float_as_int(fmaf(as, Tc[d], magic)));
      acc = min(acc, ~old & mask);
      return;
    }
    float tm2 = 1.f, tm1 = y;
    atomicAdd(&Ga[p], __float_as_int(fmaf(as, 1.f, magic)));
    atomicAdd(&Ga[W + p], __float_as_int(fmaf(as, y, magic)));
#pragma unroll
    for (int d = 2; d < kPolyChannels; d++) {
      const float t = fmaf(y2, tm1, -tm2);  // T_d = 2 y T_{d-1} - T_{d-2}
      if (d < kLast) {
        atomicAdd(&Ga[d * W + p], __float_as_int(fmaf(as, t, magic)));
      } else {
        const unsigned raw = __float_as_uint(fmaf(amp * scale_l, t, magic));
        const unsigned old = atomicAdd(reinterpret_cast<unsigned*>(&Ga[d * W + p]), raw * (1u << J) + 1u);
        acc = min(acc, ~old & mask);
      }
      tm2 = tm1;
      tm1 = t;
    }
    return;
  }
  const double yd = (double)y, y2 = 2.0 * yd, ad = (double)amp * (double)scale;
  const double magic = 6755399441055744.0;  // 1.5 2^52: the low 32 bits of (v + magic) hold round(v)
  double T[kPolyD];
  T[0] = 1.0;
  T[1] = yd;
#pragma unroll
  for (int d = 2; d < kPolyD; d++) T[d] = fma(y2, T[d - 1], -T[d - 2]);  // T_d = 2 y T_{d-1} - T_{d-2}
#pragma unroll
  for (int d = 0; d < kLast; d++) {
    const int v = __double2loint(fma(ad, T[d], magic));
    const int i = d * W + p;  // channel-major planes: consecutive positions are consecutive words
    atomicAdd(&Ga[i], v >> 14);
    atomicAdd(&Gb[i], v & 0x3FFF);
  }
  const int i = kLast * W + p;
  atomicAdd(&Ga[i], __double2loint(fma(ad * 6.103515625e-05, T[kLast], magic)));  // round(v 2^-14)
  const unsigned old = atomicAdd(reinterpret_cast<unsigned*>(&Gb[i]), 1u);
  acc = min(acc, ~old & mask);
}

// Tile format: channel resolution `bits`, one or two words, count capacity 2^J per position (jcap > 0 lowers J:
// a test hook that makes the guard fire).
__device__ __forceinline__ void poly_set_format(PolyTile& T, int bits, int two_word, int jcap) {
  T.bits = bits;
  T.two_word = two_word;
  T.scalef = ldexpf(1.f, bits - T.e);
  T.inv_scale = ldexp(1.0, T.e - bits);
  T.inv_scalef = ldexpf(1.f, T.e - bits);
  int J = two_word ? 17 : 31 - bits;
  if (jcap > 0 && jcap < J) J = jcap;
  T.J = J;
  T.cnt_mask = (1u << J) - 1u;
  T.scale_lf = ldexpf(1.f, bits - T.e - J);
}

// Plane stride W (words) fixed at compile time for ntaps <= 64 (fs <= 16 kHz at T_w = 4 ms): the 8 channel
// updates of an image and the FIR's paired-channel loads then address G with immediate offsets
__host__ __device__ constexpr int poly_plane_words(int ntaps) {
  return ((kPolyTC + ntaps - 1) + ((kPolyTC + ntaps - 1) >> 3) + 1 + 3) & ~3;  // 16-B aligned planes
}
constexpr int kPolyWFixTaps = 64;
constexpr int kPolyWFix = poly_plane_words(kPolyWFixTaps);
constexpr int kPolyMaxNear = 24;  // rotated near channels' tap window (abi.cu poly_fir_tables: 8, or 16-24 for > 64 taps)
// floats of the FIR tables in shared memory (reading R13): far [2][ntaps][2], near [2][nn][2], Q [2][4][4]
__host__ __device__ constexpr int poly_tab_floats(int ntaps, int nn) { return 4 * ntaps + 4 * nn + 32; }

// Channel rotation of reading R13 (G' = Q G, per parity): one rotated value from the four same-parity channel
// values a, b, c, d (channels par, 2 + par, 4 + par, 6 + par) — one fixed FMA order, shared by every path that
// converts G (persistent and cluster items give the same bits)
__device__ __forceinline__ float poly_rot1(const float* q, float a, float b, float c, float d) {
  return fmaf(q[3], d, fmaf(q[2], c, fmaf(q[1], b, q[0] * a)));
}
// the same for two positions at once (FMUL2 / FFMA2: each lane rounds exactly as poly_rot1)
__device__ __forceinline__ float2 poly_rot2(const float* q, float2 a, float2 b, float2 c, float2 d) {
  const float2 q0 = make_float2(q[0], q[0]), q1 = make_float2(q[1], q[1]), q2 = make_float2(q[2], q[2]),
               q3 = make_float2(q[3], q[3]);
  return __ffma2_rn(q3, d, __ffma2_rn(q2, c, __ffma2_rn(q1, b, __fmul2_rn(q0, a))));
}

// One FIR item (reading R13): outputs t8 .. t8 + 7 of partial pi = 2 s + h — the far channel pair s (rotated
// channels 2 s, 2 s + 1) over tap half h of its ntaps taps, then the near pair s (channels 4 + 2 s, 5 + 2 s) over
// half h of its nn taps — with a sliding register window, FFMA2 over the taps in order.  Gf: fp32 rotated planes
// of stride W, position p at p + p / 8, the item's first output at position ntaps - 1 (t8 relative to it).
__device__ __forceinline__ void poly_fir_range(const float* G0, int W, const float4* P4, int q, int ngroups,
                                               float2 (&acc)[8]) {
  float2 w[8];
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const int a = (q + r) + ((q + r) >> 3);
    w[r] = make_float2(G0[a], G0[a + W]);
  }
  const float* gn = G0 + (q - 1) + ((q - 1) >> 3);  // padded address of position q - 1 (= 6 mod 8)
  for (int gi = 0; gi < ngroups; gi++, gn -= 9, P4 += 4) {
    const float4 pq[4] = {P4[0], P4[1], P4[2], P4[3]};  // 8 taps of the pair, (2i, 2i + 1) per float4
#pragma unroll
    for (int u = 0; u < 8; u++) {  // tap u: output r uses slot (r - u) & 7, then slot (7 - u) & 7 refills
      const float2 pc = (u & 1) ? make_float2(pq[u >> 1].z, pq[u >> 1].w) : make_float2(pq[u >> 1].x, pq[u >> 1].y);
#pragma unroll
      for (int r = 0; r < 8; r++) acc[r] = __ffma2_rn(pc, w[(r - u) & 7], acc[r]);
      const int o = u < 7 ? -u : -8;  // the last group's refills read padding: never used
      w[(7 - u) & 7] = make_float2(gn[o], gn[o + W]);
    }
  }
}
template <bool kNear8>
__device__ __forceinline__ void poly_fir_item(const float* Gf, int W, const float* Pt, int ntaps, int nmi0, int nn,
                                              int pi, int t8, float (&res)[8]) {
  const int s = pi >> 1, h = pi & 1;
  float2 acc[8];
#pragma unroll
  for (int r = 0; r < 8; r++) acc[r] = make_float2(0.f, 0.f);
  {  // far pair s: tap groups [g0, g1) of ntaps / 8
    const int ng = ntaps >> 3, gh = (ng + 1) >> 1, g0 = h ? gh : 0, g1 = h ? ng : gh;
    const float4* P4 = reinterpret_cast<const float4*>(Pt) + s * (ntaps >> 1) + g0 * 4;
    poly_fir_range(Gf + (2 * s) * W, W, P4, t8 + ntaps - 1 - 8 * g0, g1 - g0, acc);
  }
  if constexpr (!kNear8) {  // tables of > 64 taps: the near pair's aligned window, tap groups [g0, g1) of nn / 8
    const int ng = nn >> 3, gh = (ng + 1) >> 1, g0 = h ? gh : 0, g1 = h ? ng : gh;
    const float4* P4 = reinterpret_cast<const float4*>(Pt + 4 * ntaps) + s * (nn >> 1) + g0 * 4;
    poly_fir_range(Gf + (4 + 2 * s) * W, W, P4, t8 + ntaps - 1 - nmi0 - 8 * g0, g1 - g0, acc);
  } else if (h == 0) {  // near pair s: its window's 8 taps mi = nmi0 .. nmi0 + 7 (any alignment: runtime refills)
    const float* G0 = Gf + (4 + 2 * s) * W;
    const float4* P4 = reinterpret_cast<const float4*>(Pt + 4 * ntaps) + s * (nn >> 1);
    const int q = t8 + ntaps - 1 - nmi0;  // position of output t8 at the window's first tap
    float2 w[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      const int a = (q + r) + ((q + r) >> 3);
      w[r] = make_float2(G0[a], G0[a + W]);
    }
    const float4 pq[4] = {P4[0], P4[1], P4[2], P4[3]};
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const float2 pc = (u & 1) ? make_float2(pq[u >> 1].z, pq[u >> 1].w) : make_float2(pq[u >> 1].x, pq[u >> 1].y);
#pragma unroll
      for (int r = 0; r < 8; r++) acc[r] = __ffma2_rn(pc, w[(r - u) & 7], acc[r]);
      if (u < 7) {
        const int pn = q - 1 - u, a = pn + (pn >> 3);
        w[(7 - u) & 7] = make_float2(G0[a], G0[a + W]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 8; r++) res[r] = acc[r].x + acc[r].y;
}

// CL = false: persistent CTAs taking (RIR, tile) items from a queue (large calls).  CL = true (small calls): a
// thread-block cluster of S CTAs per item — rank r aggregates the tile's columns r, r + S, ... into its own G,
// the ranks' integer G planes are summed through distributed shared memory (exactly the single CTA's sums), and
// rank r filters outputs [r 1024/S, (r + 1) 1024/S) with the same per-output arithmetic: bit-identical RIRs for
// any call size.
template <int THREADS, int WFIX, bool CL>
__global__ void __launch_bounds__(THREADS, PolyCfg<THREADS>::kCtasPerSm)
    ism_poly_kernel(IsmArgs A, long long n_work, int* work_counter) {
  using C = PolyCfg<THREADS>;
  int S = 1, rank = 0;
  if constexpr (CL) {
    S = (int)cg::this_cluster().num_blocks();
    rank = (int)cg::this_cluster().block_rank();
  }
  constexpr int kPolyThreads = C::kThreads, kPolyCols = C::kCols, kPolyGroup = C::kGroup, kPolyPass = C::kPass,
                kPolyPasses = C::kPasses;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PolySmem<THREADS>& sm = *reinterpret_cast<PolySmem<THREADS>*>(smem_raw);
  const int ntaps = A.poly_ntaps, npos = kPolyTC + ntaps - 1;
  (void)npos;  // the cluster branch uses its item's own count
  // channel planes of W words, position p at p + p/8: the filter's lanes read positions 8 apart, which the
  // padding spreads over all banks (stride 9 words)
  const int W = WFIX > 0 ? WFIX : poly_plane_words(ntaps);
  int* Ga = reinterpret_cast<int*>(smem_raw + sizeof(PolySmem<THREADS>));  // coarse part of G (units 2^14)
  int* Gb = Ga + kPolyD * W;                                       // fine part of G (two-word calls only)
  float* Pt = reinterpret_cast<float*>(Gb + (A.poly_gb ? kPolyD * W : 0));        // [4 pairs][ntaps][2], mi = m - m_lo
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double fs_over_c = A.fs_over_c, sc2 = fs_over_c * fs_over_c;
  const float fs_over_c_4pi = (float)fs_over_c * 0.0795774715459476679f, fsc = (float)fs_over_c;
  const int m_hi = A.poly_mlo + ntaps - 1;
  constexpr int kLast = kPolyChannels - 1;  // the channel whose word also counts (poly_add)

#ifdef GPURIR_PHASE_TIMING
  unsigned long long pt_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pts_[5] = {0, 0, 0, 0, 0};
  unsigned long long ptl_[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pta_[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  PT_MARK(0);
  PS_MARK(0);
  if constexpr (CL) {  // small calls: threads >= 32 copy the table, thread 0 goes straight to its item's setup
    if (tid >= 32)
      for (int i = tid - 32; i < poly_tab_floats(ntaps, A.poly_nn); i += kPolyThreads - 32) Pt[i] = A.poly_P[i];
  } else {
    for (int i = tid; i < poly_tab_floats(ntaps, A.poly_nn); i += kPolyThreads) Pt[i] = A.poly_P[i];
  }
  // (the FIR window nmi0 / nn and the rotation Q = Pt + 4 ntaps + 4 nn are re-read from the parameter bank where
  // used: no registers held across the image loop)
  PS_MARK(1);
  if (tid == 0) sm.pf_valid = 0;  // read by thread 0 only, after the loop top's barrier
  bool bz_ready = false;          // sm.bz holds this call's z factors (single-room calls)

  for (;;) {
    PTL_MARK(0);
    if (tid >= 32) {  // zero G while thread 0 sets the next work item up (G is free: the loop ends in a barrier)
      // 16-B stores over the 8 W words of each array
      const int n4 = (kPolyD * W) >> 2;
      const bool both = A.poly_gbz;  // the call has two-word tiles: zero the fine plane with the coarse one
      for (int i = tid - 32; i < n4; i += kPolyThreads - 32) reinterpret_cast<int4*>(Ga)[i] = make_int4(0, 0, 0, 0);
      if (both)
        for (int i = tid - 32; i < n4; i += kPolyThreads - 32) reinterpret_cast<int4*>(Gb)[i] = make_int4(0, 0, 0, 0);
      // a single-room call's z-factor table depends only on the call's arguments: built here, beside thread 0's
      // setup, instead of after it (the cluster items of small calls build it for their one item: -0.5 us)
      if (!A.jobs && !bz_ready && A.nb[2] <= kPolyBz)
        for (int i = tid - 32; i < A.nb[2]; i += kPolyThreads - 32) sm.bz[i] = poly_z_factor_args(i - A.nb[2] / 2, A);
    } else if (tid == 0) {
      long long wi;
      int sub = 0, nsub = 1;  // this cluster's output sub-range of the item, of nsub
      long long w;  // the call's work entry: a cluster, or the queue's next entry
      if (CL) {
        w = (long long)(blockIdx.x / S);
      } else if (sm.pf_valid) {  // prefetched during the previous item's filter
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        w = sm.pf_wi;
      } else {
        w = atomicAdd(work_counter, 1);
      }
      PolyTile& T = sm.ti;
      if (CL) {  // every cluster has an entry; n_work counts items
        wi = poly_decode(A, w, sub, nsub);
        T.next = wi < n_work;
      } else if constexpr (THREADS >= 512) {  // n_work counts queue entries (split plans: calls of <= 2 items per SM)
        T.next = w < n_work;
        wi = T.next ? poly_decode(A, w, sub, nsub) : w;  // the item and this entry's output sub-range
      } else {   // 256- and 512-thread CTAs: one entry per item
        T.next = w < n_work;
        wi = w;
      }
      PS_MARK(2);
      if (wi < n_work) {
        int m, tile, nISM;
        long long row;
        const float zero3[3] = {0.f, 0.f, 0.f};
        if (A.jobs) {
          const int2 jt = A.tiles[wi];
          const BatchJob& J = A.jobs[jt.x];
          m = jt.x; tile = jt.y; nISM = J.nISM; row = J.out_offset;
          geom_from(J.L, J.src, J.rcv, J.orv, J.nb, J.pattern, J.ors, J.spkr_pattern, J.lb, J.neg, J.zero, T.g,
                    A.status);
        } else {
          long long rm;
          tile = A.nTiles - 1 - (int)poly_divmod(wi, A.M, A.invM, rm);  // heaviest (latest) tiles first
          m = (int)rm;
          nISM = A.nISM;
          row = (long long)m * A.row_stride;
          long long mr;
          const int ms = (int)poly_divmod(m, A.M_rcv, A.invMrcv, mr);
          if (!CL && sm.pf_valid)  // the inputs were fetched with the index
            geom_from(A.L, sm.pf_in, sm.pf_in + 3, A.orv ? sm.pf_in + 6 : zero3, A.nb, A.pattern,
                      A.ors ? sm.pf_in + 9 : zero3, A.spkr_pattern, A.lb, A.neg, A.zero, T.g, A.status);
          else if constexpr (CL) {  // small calls: all 12 inputs in flight at once (geom_from stores into shared
                                    // memory, which the compiler must assume the input pointers alias)
            float in[12];
#pragma unroll
            for (int k = 0; k < 3; k++) {
              in[k] = A.pos_src[3 * ms + k];
              in[3 + k] = A.pos_rcv[3 * mr + k];
              in[6 + k] = A.orv ? A.orv[3 * mr + k] : 0.f;
              in[9 + k] = A.ors ? A.ors[3 * ms + k] : 0.f;
            }
            geom_from(A.L, in, in + 3, in + 6, A.nb, A.pattern, in + 9, A.spkr_pattern, A.lb, A.neg, A.zero, T.g,
                      A.status);
          } else
            geom_from(A.L, A.pos_src + 3 * ms, A.pos_rcv + 3 * mr, A.orv ? A.orv + 3 * mr : zero3, A.nb, A.pattern,
                      A.ors ? A.ors + 3 * ms : zero3, A.spkr_pattern, A.lb, A.neg, A.zero, T.g, A.status);
        }
        T.row = row;
        T.rir = m;
        PS_MARK(3);
        // tiles end-aligned ([nISM - 1024 (k + 1), nISM - 1024 k)), so the last one holds the whole envelope
        // window when the tail is fused; also when it is not, because the fixed-point scale is per tile and a RIR
        // must give the same bits whether or not its tail is fused (shards of one call fuse or not by size), and
        // the same bits in a batch of rooms as alone
        const int ntile = (nISM + kPolyTC - 1) / kPolyTC;
        T.te = nISM - (ntile - 1 - tile) * kPolyTC;
        T.t0 = max(0, T.te - kPolyTC);
        // the item's outputs: sub-range `sub` of nsub equal end-aligned parts (nsub > 1 only for full tiles; the
        // fixed-point format below stays the whole tile's); positions cover the nominal part + the halo
        {  // parts of Ls outputs, a multiple of 128 (so a cluster rank's share stays a multiple of 8 for S <= 16):
           // 1024 / nsub for a full tile; a partial (first) tile's first part takes what is left
          const int Ls = nsub > 1 ? (((T.te - T.t0 + nsub - 1) / nsub + 127) & ~127) : kPolyTC;
          T.ote = T.te - (nsub - 1 - sub) * Ls;
          T.ot0 = nsub > 1 ? max(T.t0, T.ote - Ls) : T.t0;
          T.npos_i = Ls + ntaps - 1;
        }
        if (A.jobs) {
          const BatchJob& J = A.jobs[m];
          T.tail = A.poly_tail && tile == ntile - 1 && J.nISM < J.nS;
          T.tail_nS = J.nS;
          T.tail_kappa = J.kappa_fs;
          T.tail_rglob = J.rir_global;
        } else {
          T.tail = A.poly_tail && tile == ntile - 1 && sub == nsub - 1;
          T.tail_nS = A.tail_nS;
          T.tail_kappa = A.tail_kappa_fs;
          T.tail_rglob = A.tail_rir_base + (unsigned long long)m;
        }
        T.tc = T.t0 + kPolyTC / 2;
        const double* geo = A.jobs ? A.jobs[m].geo : A.poly_geo;  // 1/L, 1/V_s, 1/L_min,s (host reciprocals)
        T.invLz = geo[2];
        T.Lzs = T.g.L[2] * A.fs_over_c;
        T.offEs = (T.g.s[2] - T.g.r[2]) * A.fs_over_c;
        T.offOs = (-T.g.s[2] - T.g.r[2]) * A.fs_over_c;
        // images with floor(x) in [t0 - m_hi, te - 1 - m_lo] reach samples [t0, te)
        const double xlo = (double)(T.ot0 - m_hi), xhi = (double)(T.ote - A.poly_mlo);  // this item's shell
        const double dlo = xlo > 0.0 ? xlo * A.c_over_fs : 0.0, dhi = xhi * A.c_over_fs;
        T.dlo2 = dlo * dlo;
        T.dhi2 = dhi * dhi;
        int lo[2], hi[2];
        for (int ax = 0; ax < 2; ax++) {
          const double iL = geo[ax], r = T.g.r[ax];  // the -1 / +1 margins cover the reciprocal's rounding
          const int a = (int)floor((r - dhi) * iL) - 1, b = (int)floor((r + dhi) * iL) + 1;
          lo[ax] = max(a, T.g.nlo[ax]);
          hi[ax] = min(b, T.g.nhi[ax] - 1);
        }
        T.nx0 = lo[0]; T.ny0 = lo[1];
        T.NX = max(0, hi[0] - lo[0] + 1);
        T.ncols = T.NX * max(0, hi[1] - lo[1] + 1);
        T.invNX = T.NX > 0 ? 1.f / (float)T.NX : 0.f;
        T.zl = T.g.nlo[2];
        T.zh = T.g.nhi[2] - 1;
        T.use_bz = (T.zh - T.zl + 1) <= kPolyBz;
        // per-tile fixed point (see poly_add).  Images depositing into this tile have x >= x_lo =
        // max(t0 - m_hi, x_dp) samples (the direct path is the closest image), so |A_n| <= 1 / (4 pi d_lo)
        // (|beta|, |g| <= 1) and every channel value is |v| <= 2^bits.  The resolution is chosen from an
        // ESTIMATE N of the images sharing one sample position at delays <= x_hi (the tile's largest): twice the
        // mean count 4 pi x_hi^2 / V_s (one image per room volume V_s, in samples), plus 24 x_hi / (L_min fs / c)
        // for images stacked on equal distances by symmetric or commensurate geometry, plus 16;
        // bits = min(22, 30 - ceil(log2 N)), i.e. a count capacity 2^(31 - bits) > 2N.  N is a heuristic (the
        // number of lattice points on a sphere is not bounded by any fixed multiple of the mean: DESIGN.md
        // §5.5); correctness rests on the exact count guard of poly_add, which redoes a tile whose capacity is
        // reached.  Below 18 bits (N >= 2^12) the tile takes the two-word scheme: single-word tiles keep
        // 2 bits - 31 >= 5 bits for the counting channel (poly_add).
        const double ddx = T.g.s[0] - T.g.r[0], ddy = T.g.s[1] - T.g.r[1], ddz = T.g.s[2] - T.g.r[2];
        const double x_dp = sqrt(ddx * ddx + ddy * ddy + ddz * ddz) * A.fs_over_c;
        T.x_dp = x_dp;
        const double x_lo = fmax(fmax((double)(T.t0 - m_hi), x_dp), 1e-30);
        const double x_hi = (double)(T.te - A.poly_mlo);
        int lb;
        (void)frexp(25.132741228718345 * x_hi * x_hi * geo[3] + 24.0 * x_hi * geo[4] + 16.0, &lb);  // N < 2^lb
        int bits = min(22, 30 - lb);
        const int two_word = bits < 18 || A.poly_force2 || A.poly_hook == 3;
        if (two_word) bits = 28;
        const double abound = 0.0795774715459476679 * A.fs_over_c / x_lo;
        (void)frexp(abound, &T.e);  // abound < 2^e
        poly_set_format(T, bits, two_word, A.poly_hook >= 2 ? 2 : 0);
        T.ovf = 0;
      }
    }
    PS_MARK(4);
    __syncthreads();
    if (!sm.ti.next) { PTL_DUMP(); break; }
    PT_MARK(1);
    PTL_MARK(1);
    const PolyTile& T = sm.ti;
    const RirGeom& g = T.g;
    // the z factors depend only on the room: once per CTA for a single-room call, per item for a batch of rooms
    // (single-room calls with nb_z <= kPolyBz: built before the barrier above, T.zl = -(nb_z / 2))
    if (T.use_bz && (A.jobs || !(bz_ready || A.nb[2] <= kPolyBz)))
      for (int i = tid; i <= T.zh - T.zl; i += kPolyThreads) sm.bz[i] = poly_z_factor(T.zl + i, g);
    bz_ready = true;

    PT_MARK(2);
    PTL_MARK(2);
    // ---- 1. image aggregation -------------------------------------------------------------
    // Redone (once) when the count guard fires: a single-word tile goes to the two-word format (capacity 2^17
    // images per position) if the call's shared memory holds the fine plane; otherwise — and for a two-word
    // tile that fires — the capacity status is set instead of returning a wrapped sum.  The format
    // depends only on this tile's own images (deterministic, shard-invariant; a call launched without the fine
    // plane, i.e. 256-thread CTAs, reports the capacity status where a 512-thread call would go on).
    for (;;) {
      const float amp_scale = fs_over_c_4pi;
      const int pbase = sm.ti.ot0 - m_hi;  // p = floor(x) - pbase
      const int npos_i = sm.ti.npos_i;
      const int ncl = CL ? (T.ncols - rank + S - 1) / S : T.ncols;  // this rank's columns: rank, rank + S, ...
      for (int qb = 0; qb < ncl; qb += kPolyCols) {
        int cnt = 0;
        {
          const int q = CL ? (qb + tid) * S + rank : qb + tid;
          PolyColRec cr;
          cr.a1 = 0; cr.a2 = 0; cr.b = 0; cr.end = 0; cr.rho2 = 0.0; cr.bxy = 0.f; cr.cdot = 0.f;
          float sdot = 0.f;
          int r1lo = 0, r2lo = 0, r1n = 0;
          if (q < T.ncols) {
            const int qy = (int)(((float)q + 0.5f) * T.invNX);
            const int nx = T.nx0 + (q - qy * T.NX), ny = T.ny0 + qy;
            const double dx = image_coord(nx, g.L[0], g.s[0]) - g.r[0];
            const double dy = image_coord(ny, g.L[1], g.s[1]) - g.r[1];
            const double rho2 = dx * dx + dy * dy;
            cr.rho2 = rho2 * sc2;
            cr.cdot = ((float)dx * g.o[0] + (float)dy * g.o[1]) * fsc;
            sdot = src_col_dot(nx, ny, (float)dx, (float)dy, g) * fsc;
            uint32_t sgn = 0;
            bool zero = false;
            const float lxy = axis_beta(nx, 0, g, sgn, zero) + axis_beta(ny, 1, g, sgn, zero);
            const float bxy = zero ? 0.f : ex2_approx(lxy);
            cr.bxy = (sgn ? -bxy : bxy) * amp_scale * T.scalef;  // the tile's fixed-point scale (a power of two) folded in
            if (rho2 < T.dhi2) {
              const double zhi = (double)sqrtf((float)(T.dhi2 - rho2));
              const double zlo = T.dlo2 > rho2 ? (double)sqrtf((float)(T.dlo2 - rho2)) : 0.0;
              int pa, pb, na, nbz;
              z_range(g, T.invLz, zlo, zhi, pa, pb);
              z_range(g, T.invLz, -zhi, -zlo, na, nbz);
              if (nbz >= pa - 1) { pa = min(pa, na); na = 1; nbz = 0; }
              pa = max(pa, T.zl); pb = min(pb, T.zh);
              na = max(na, T.zl); nbz = min(nbz, T.zh);
              const int n1 = max(0, pb - pa + 1), n2 = max(0, nbz - na + 1);
              r1lo = pa; r1n = n1; r2lo = na;
              cnt = n1 + n2;
              if (rho2 == 0.0 && cnt > 0) {  // an image on the receiver (x2 = 0, Eq. 2 degenerate): the column says so
                const double zr = g.r[2], zs = g.s[2], Lz = g.L[2];
                const int ce = 2 * (int)rint((zr - zs) / (2.0 * Lz)), co = 2 * (int)rint((zr + zs) / (2.0 * Lz)) - 1;
                for (int c2 = 0; c2 < 2; c2++) {
                  const int nzc = c2 ? co : ce, nzo = nzc + (nzc & 1);
                  const bool in = (nzc >= pa && nzc < pa + n1) || (nzc >= na && nzc < na + n2);
                  if (in && fma(int_to_double(nzo), T.Lzs, (nzc & 1) ? T.offOs : T.offEs) == 0.0)
                    atomicOr(A.status, kStatusDegenerate);
                }
              }
            }
          }
          // one scan of (candidates + 2^20 x nonempty) both prefixes the candidates and compacts the nonempty
          // columns in order, so the run search and the walk below never visit an empty column
          const int incl = poly_block_scan<kPolyThreads>(cnt + (cnt > 0 ? (1 << 20) : 0), sm.scan_tmp);
          if (cnt > 0) {
            const int end = incl & 0xFFFFF, start = end - cnt, k = (incl >> 20) - 1;
            cr.end = end;
            cr.b = start + r1n;          // first candidate of the second n_z run
            // n_z + 2^31 = gi + a1 on the first run, gi + a2 on the second (mod 2^32): the walk forms the
            // exponent-bias bits of its int -> double conversion directly
            cr.a1 = (int)((unsigned)(r1lo - start) + 0x80000000u);
            cr.a2 = (int)((unsigned)(r2lo - r1n - start) + 0x80000000u);
            sm.col[k] = cr;
            sm.colpre[k] = end;
            sm.colsdot[k] = sdot;
          }
        }
        __syncthreads();
        const int tot = sm.scan_tmp[kPolyThreads / 32 - 1];
        const int total = tot & 0xFFFFF, ncomp = tot >> 20;
        const int R = (total + kPolyThreads - 1) / kPolyThreads;
        const int g0 = tid * R, g1 = min(g0 + R, total);
        if (g0 < g1) {
          int lo = 0, hi = ncomp - 1;  // first (compacted) column with colpre > g0
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm.colpre[mid] > g0) hi = mid; else lo = mid + 1;
          }
          int j = lo;
          const int zl = T.zl;
          const unsigned zlb = (unsigned)zl + 0x80000000u;
          // the column records carry the fixed-point scale, so the deposits take amp as is and the last channel
          // amp 2^-J (both exact: powers of two)
          const float oz = g.o[2], ga = g.a, oma = 1.f - ga, scale_lj = T.scale_lf / T.scalef;
          const int J = T.J;
          const unsigned cmask = T.cnt_mask;
          unsigned acc = 0xFFFFFFFFu;  // min of ~old & mask over this thread's last-channel deposits (poly_add)
          PolyColRec cr = load_col(&sm.col[j]);  // the current column's record, in registers
          // the walk, compiled three times: the common case (single word, omni source, z factors from the table)
          // with its flags as constants — fewer live registers, so fewer loop constants re-read from shared memory —
          // once more for single-room calls on 256-thread CTAs (pattern constants from the parameter bank: +0.2 %), and the
          // general case with runtime flags
          auto walk = [&](auto fast, auto single) {
          constexpr bool kFast = decltype(fast)::value, kSingle = decltype(single)::value;
          // single-room calls: the receiver pattern's constants straight from the parameter bank (uniform registers,
          // off the 64-register budget of the loop)
          const float gaw = kSingle ? pattern_const(A.pattern) : ga, omaw = kSingle ? 1.f - pattern_const(A.pattern) : oma;
          const bool use_bz = kFast || T.use_bz, dir_src = !kFast && g.as != 1.f, two_word = !kFast && T.two_word;
          const double Lzs = T.Lzs, offEs = T.offEs, offOs = T.offOs;
          for (int gi = g0; gi < g1; gi++) {  // every lane runs R candidates: the walk keeps the warp converged
            // compacted columns are nonempty and gi advances by one: a change moves exactly one column on
            if (gi >= cr.end) cr = load_col(&sm.col[++j]);
            const unsigned nzb = (unsigned)gi + (unsigned)(gi < cr.b ? cr.a1 : cr.a2);  // n_z + 2^31
            const int odd = (int)(nzb & 1u);
            // nz lies in [zl, zh] (the column's runs are clamped to it) and use_bz means zh - zl < kPolyBz
            const float bz = use_bz ? sm.bz[nzb - zlb] : poly_z_factor((int)(nzb - 0x80000000u), g);
            const unsigned nzob = nzb + (unsigned)odd;
            // Eq. 1 along z, in samples: (2^52 + 2^31 + n_zo) as raw bits minus 2^52 + 2^31 (int_to_double)
            const double dz = fma(__hiloint2double(0x43300000, (int)nzob) - A.poly_i2d_bias, Lzs, odd ? offOs : offEs);
            const double x2 = fma(dz, dz, cr.rho2);                             // (d fs / c)^2

            float x0f, xd, rx;  // x = x0f + xd (xd the fp64 Newton correction); rx = 1/x
            delay_split(x2, x0f, xd, rx);
            // floor of x0f (exact: x0f is a float), fraction (x0f - floor) + xd, then one step back or forward when
            // xd carries the fraction out of [0, 1) (|xd| <= 2.4e-7 x).  Flooring the fp32 SUM x0f + xd instead
            // picks the wrong integer within half an fp32 ulp of x (5e-4 samples at x ~ 1.3e4) and the clamp then
            // moves phi by that much: harmless for one image, 1.7e-4 of peak for the ~500 images a rigid centred
            // cube stacks on one delay at 48 kHz (tests/test_gpu_parity.py::test_poly_worst_geometry_found)
            int jfl;
            const float fj = floor_int(x0f, jfl);
            float phi = (x0f - fj) + xd;
            {  // phi in (-1, 2): one more exact floor moves it into [0, 1) (5 instructions instead of the 9 of a
               // compare-and-select fix-up: +0.8 %).  An image at the receiver (x2 = 0, flagged by its column above)
               // gives a NaN delay, whose floors' integer bits put p far out of range: it is dropped below.
              int k;
              phi -= floor_int(phi, k);
              jfl += k;
            }
            phi = fminf(phi, 0.99999994f);  // phi + 1 rounds to 1 for phi > -3e-8
            const int p = jfl - pbase;
            if ((unsigned)p >= (unsigned)npos_i) continue;  // reaches no sample of this item (p < 0 wraps)
            const float dzf = (float)dz;  // one XU conversion instead of shared-memory loads (the smem pipe binds)
            const float cth = fmaf(dzf, oz, cr.cdot) * rx;
            float gain = fmaf(omaw, cth, gaw);
            if (dir_src) gain *= src_gain(sm.colsdot[j], odd, dzf, rx, g);
            const float amp = cr.bxy * bz * gain * rx;       // Eq. 4
            const float y = fmaf(2.f, phi, A.poly_m1);        // 2 phi - 1 in [-1, 1)
            // (cluster items keep the original deposit order: their code is tuned for latency, measured separately)
            poly_add<!CL>(Ga, Gb, W, p + (p >> 3), y, amp, 1.f, scale_lj, J, cmask, two_word, acc);
          }
          };
          if (T.use_bz && !T.two_word && g.as == 1.f) {
            // (256-thread CTAs only: in the 512-thread variant the extra instantiation cost config 4 8 %)
            if (!CL && THREADS == 256 && !A.jobs) walk(std::true_type(), std::true_type());
            else walk(std::true_type(), std::false_type());
          } else {
            walk(std::false_type(), std::false_type());
          }
          if (acc == 0u) sm.ti.ovf = 1;  // a position of this tile reached its count capacity
        }
        __syncthreads();  // column records are replaced by the next batch
      }
      const int ovf = sm.ti.ovf;  // read after the last batch's barrier; uniform
      PT_MARK(3);
      PTL_MARK(3);
      if (CL || !ovf) break;      // cluster items check the summed counts below (no redo: capacity status)
      __syncthreads();  // everyone has read the flag before thread 0 changes the format
      if (tid == 0) {
        PolyTile& Tw = sm.ti;
        Tw.ovf = 0;
        Tw.redo = 1;
        if (!Tw.two_word && A.poly_gb) {
          poly_set_format(Tw, 28, 1, 0);
        } else {
          atomicOr(A.status, kStatusCapacity);
          Tw.redo = 0;
        }
      }
      __syncthreads();
      if (!sm.ti.redo) break;
      {
        const int n4 = (kPolyD * W) >> 2;
        for (int i = tid; i < n4; i += kPolyThreads) reinterpret_cast<int4*>(Ga)[i] = make_int4(0, 0, 0, 0);
        if (sm.ti.two_word)
          for (int i = tid; i < n4; i += kPolyThreads) reinterpret_cast<int4*>(Gb)[i] = make_int4(0, 0, 0, 0);
      }
      __syncthreads();
    }

    if constexpr (CL) {
      // ---- 2'. cluster: sum the ranks' integer planes over DSMEM for this rank's positions, fp32, FIR -------
      cg::cluster_group cl = cg::this_cluster();
      const int npos = T.npos_i;  // this item's positions (its nominal outputs + the halo)
      const int R = (npos - ntaps + 1) / S, o0 = rank * R, npp = R + ntaps - 1;  // outputs and positions of this rank
      // The ranks' integer planes meet through L2 (distributed shared memory moves only ~20 B per clock per SM: a
      // pull of the ranks' planes, or a push of their words by DSMEM reductions into the owners, measured 2x slower):
      // (1) every rank stores its planes to its slab; (2) each rank sums a disjoint range of Pq positions over the
      // ranks' slabs (integer sums mod 2^32: exactly the single-CTA G) and converts them to fp32 in its staging area;
      // (3) each rank gathers the positions its FIR needs — its R outputs plus the halo — from the owners (DSMEM).
      const int Ws = A.poly_slab_w;                     // slab plane stride (words, >= npos)
      const int nw = T.two_word ? 2 * kPolyD : kPolyD;  // integer planes: coarse, then fine
      const size_t slab_words = (size_t)2 * kPolyD * Ws;
      const unsigned* slab0 = A.poly_slab + (size_t)(blockIdx.x - rank) * slab_words;  // this cluster's rank 0
      {
        unsigned* my = A.poly_slab + (size_t)blockIdx.x * slab_words;
        const unsigned* Gu = reinterpret_cast<const unsigned*>(Ga);  // Gb follows Ga at kPolyD W words
        for (int i = tid; i < nw * npos; i += kPolyThreads) {
          const int d = i / npos, p = i - d * npos;
          __stcg(&my[(size_t)d * Ws + p], Gu[d * W + p + (p >> 3)]);
        }
      }
      cl.sync();  // barrier.cluster arrive.release / wait.acquire: every rank's slab stores are visible
      PT_MARK(4);
      const int Pq = (npos + S - 1) / S, q0 = rank * Pq, nq = max(0, min(npos, q0 + Pq) - q0);
      unsigned* stu = reinterpret_cast<unsigned*>(Ga);      // [nw][Pq] sums, then [Pq] counts (G is free now)
      float* stf = reinterpret_cast<float*>(sm.col);        // [kPolyD][Pq] fp32 totals, read by the other ranks
      const unsigned cmask = T.two_word ? 0u : T.cnt_mask;
      for (int i = tid; i < nw * nq; i += kPolyThreads) {
        const int d = i / nq, pi = i - d * nq;
        const unsigned* src = slab0 + (size_t)d * Ws + q0 + pi;
        unsigned x[16], w = 0u, n = 0u;  // S = 4, 8 or 16: all S loads in flight at once
#pragma unroll
        for (int u = 0; u < 16; u++) x[u] = u < S ? __ldcg(src + (size_t)u * slab_words) : 0u;
#pragma unroll
        for (int u = 0; u < 16; u++) { w += x[u]; n += x[u] & cmask; }  // counts sum without wrapping
        stu[d * Pq + pi] = w;
        if (d == kLast) stu[nw * Pq + pi] = n;
      }
      __syncthreads();
      {
        bool bad = tid == 0 && T.ovf;  // this rank's own guard fired
        const unsigned kLastOff = 1u + (0x4B400000u << T.J);
        for (int pi = tid; pi < nq; pi += kPolyThreads) {
          float v[kPolyD];
          if (!T.two_word) {
            const unsigned n = stu[nw * Pq + pi];
            bad = bad || n > T.cnt_mask;  // 2^J images on this position in all: as the guard
#pragma unroll
            for (int d = 0; d < kPolyD; d++) {
              const unsigned off = d < kLast ? 0x4B400000u : d == kLast ? kLastOff : 0u;
              v[d] = (float)(int)(stu[d * Pq + pi] - n * off) * T.inv_scalef;
            }
          } else {
            bad = bad || stu[(kPolyD + kLast) * Pq + pi] > T.cnt_mask;
#pragma unroll
            for (int d = 0; d < kPolyD; d++) {
              const int ca = (int)stu[d * Pq + pi], fb = (int)stu[(kPolyD + d) * Pq + pi];
              v[d] = d == kLast ? (float)((double)ca * 16384.0 * T.inv_scale)
                                : (float)((double)((long long)ca * 16384 + fb) * T.inv_scale);
            }
          }
          const float* Qr = Pt + 4 * ntaps + 4 * A.poly_nn;
#pragma unroll
          for (int par = 0; par < 2; par++)  // rotated channels (reading R13): stf holds G' = Q G
#pragma unroll
            for (int k = 0; k < 4; k++)
              stf[(2 * k + par) * Pq + pi] = poly_rot1(Qr + (par * 4 + k) * 4, v[par], v[2 + par], v[4 + par], v[6 + par]);
        }
        if (bad) atomicOr(A.status, kStatusCapacity);
      }
      cl.sync();  // every rank's totals are staged
      // the positions this rank's FIR needs, [o0, o0 + npp): its own and the halo, from the owners over DSMEM
      float* Gf = reinterpret_cast<float*>(Ga);
      for (int i = tid; i < kPolyD * npp; i += kPolyThreads) {
        const int d = i / npp, pi = i - d * npp, p = o0 + pi, own = p / Pq;
        Gf[d * W + pi + (pi >> 3)] = cl.map_shared_rank(stf, own)[d * Pq + (p - own * Pq)];
      }
      cl.sync();  // every rank has gathered: the staging areas are free
      PT_MARK(5);
      // FIR over this rank's R outputs with the persistent path's arithmetic (so the same bits): item (partial pi,
      // 8 consecutive outputs) of poly_fir_item, then per output the partials ((p0 + p1) + (p2 + p3)); all positions
      // are local to the rank (o0 is its first output)
      float* red = reinterpret_cast<float*>(sm.col);  // [4 partials][R]
      for (int it = tid; it < 4 * (R >> 3); it += kPolyThreads) {
        const int pi = it / (R >> 3), t8 = 8 * (it - pi * (R >> 3));
        float res[8];
        poly_fir_item<(WFIX > 0)>(Gf, W, Pt, ntaps, A.poly_nmi0, A.poly_nn, pi, t8, res);
#pragma unroll
        for (int r = 0; r < 8; r++) red[pi * R + t8 + r] = res[r];
      }
      __syncthreads();
      for (int o = tid; o < R; o += kPolyThreads) {
        const int k = T.ot0 + o0 + o;
        if (k < T.ote) A.out[T.row + k] = (red[o] + red[R + o]) + (red[2 * R + o] + red[3 * R + o]);
      }
      PT_MARK(6);
      if (T.tail)  // uniform over the cluster
        poly_fused_tail_cl(sm.ti, A.out + T.row, tid, A.out, A.tail_win, A.tail_seed, rank * kPolyThreads,
                           S * kPolyThreads);
      PT_MARK(7);
      PT_DUMP();
      break;  // one item per cluster (no rank reads another's shared memory)
    } else {
      // ---- 2. fixed point -> fp32, in place (every word converts itself: no staging, one barrier) ---------
      float* Gf = reinterpret_cast<float*>(Ga);
      long long wi_next = 0;
      if (tid == 0) wi_next = atomicAdd(work_counter, 1);  // the next item's index; its latency hides under the work
      // every thread converts whole positions (all 8 channels) and rotates them in place: G' = Q G (reading R13)
      const float* Qr = Pt + 4 * ntaps + 4 * A.poly_nn;
      if (T.two_word) {
        for (int p = tid; p < W; p += kPolyThreads) {
          float v[kPolyD];
#pragma unroll
          for (int d = 0; d < kPolyD; d++) {
            const int i = d * W + p;
            v[d] = d == kLast ? (float)((double)Ga[i] * 16384.0 * T.inv_scale)
                              : (float)((double)((long long)Ga[i] * 16384 + Gb[i]) * T.inv_scale);
          }
#pragma unroll
          for (int par = 0; par < 2; par++)
#pragma unroll
            for (int k = 0; k < 4; k++)
              Gf[(2 * k + par) * W + p] = poly_rot1(Qr + (par * 4 + k) * 4, v[par], v[2 + par], v[4 + par], v[6 + par]);
        }
      } else {  // single word, |sum| < 2^31: one rounding to fp32 (I2FP, ALU pipe), then an exact power-of-two scale
        // each thread owns 4 positions of every plane: it reads their counts from the last channel's low bits
        // and removes count x 0x4B400000 (the raw-bit deposits of poly_add) from every channel
        const float is = T.inv_scalef;
        const unsigned mask = T.cnt_mask, kLastOff = 1u + (0x4B400000u << T.J);
        const int w4 = W >> 2;  // W is a multiple of 4
        for (int q = tid; q < w4; q += kPolyThreads) {
          const uint4 c = reinterpret_cast<const uint4*>(Ga)[kLast * w4 + q];
          const uint4 n = make_uint4(c.x & mask, c.y & mask, c.z & mask, c.w & mask);
  #pragma unroll
          for (int par = 0; par < 2; par++) {  // one parity at a time: its 4 planes are read before any is written
            float4 v[4];
  #pragma unroll
            for (int i = 0; i < 4; i++) {
              const int d = 2 * i + par;
              const unsigned off = d < kLast ? 0x4B400000u : d == kLast ? kLastOff : 0u;  // planes past kLast stay 0
              const uint4 u = d == kLast ? c : reinterpret_cast<const uint4*>(Ga)[d * w4 + q];
              v[i] = make_float4((float)(int)(u.x - n.x * off) * is, (float)(int)(u.y - n.y * off) * is,
                                 (float)(int)(u.z - n.z * off) * is, (float)(int)(u.w - n.w * off) * is);
            }
  #pragma unroll
            for (int k = 0; k < 4; k++) {
              const float* qk = Qr + (par * 4 + k) * 4;
              const float2 lo = poly_rot2(qk, make_float2(v[0].x, v[0].y), make_float2(v[1].x, v[1].y),
                                          make_float2(v[2].x, v[2].y), make_float2(v[3].x, v[3].y));
              const float2 hi = poly_rot2(qk, make_float2(v[0].z, v[0].w), make_float2(v[1].z, v[1].w),
                                          make_float2(v[2].z, v[2].w), make_float2(v[3].z, v[3].w));
              reinterpret_cast<float4*>(Gf)[(2 * k + par) * w4 + q] = make_float4(lo.x, lo.y, hi.x, hi.y);
            }
          }
        }
      }
      __syncthreads();
      PTL_MARK(4);
      if (tid == 0) {  // the next item's inputs, asynchronously into shared memory (single-room calls)
        sm.pf_wi = wi_next;
        sm.pf_valid = 1;
        if (!A.jobs && wi_next < n_work) {
          long long rm, mr;
          int s_, n_;
          (void)poly_divmod(THREADS >= 512 ? poly_decode(A, wi_next, s_, n_) : wi_next, A.M, A.invM, rm);
          const int ms = (int)poly_divmod(rm, A.M_rcv, A.invMrcv, mr);
          for (int k = 0; k < 3; k++) {
            poly_cp4(&sm.pf_in[k], A.pos_src + 3 * ms + k);
            poly_cp4(&sm.pf_in[3 + k], A.pos_rcv + 3 * mr + k);
            if (A.orv) poly_cp4(&sm.pf_in[6 + k], A.orv + 3 * mr + k);
            if (A.ors) poly_cp4(&sm.pf_in[9 + k], A.ors + 3 * ms + k);
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      }

      // ---- 3. FIR: h[k] = sum_m sum_d P'_d[m] G'_d[k - m] (reading R13: rotated channels 0..3 over all ntaps
      // taps, 4..7 over the nn taps of their window) ------------------------------------------------------------
      // 512 items (partial pi = 2 s + h, 8 consecutive outputs), kPolyPasses per thread (poly_fir_item: a sliding
      // register window per channel pair); the 4 partial sums meet in shared memory.  ntaps is padded to a multiple of
      // 8 with zero taps, so in every unrolled group of 8 taps the new positions sit at fixed offsets 0 .. -6, -8 of
      // one padded address.
      {
        static_assert(kPolyPasses <= 2, "earlier passes' partials are parked in the column records (THREADS x 8 floats)");
        float4* park = reinterpret_cast<float4*>(sm.col);  // free during the FIR; keeps registers for the window
        float part[8];
        constexpr int kItems = 4 * (kPolyTC / 8);  // (1024-thread CTAs: threads >= kItems idle here)
        constexpr bool kIdle = kPolyThreads * kPolyPasses > kItems;
  #pragma unroll
        for (int pass = 0; pass < kPolyPasses; pass++) {
          // two passes: a thread takes partials (0, 3) or (1, 2), one with and one without the near taps
          const int it = pass * kPolyThreads + tid, pi0 = it >> 7, pi = (kPolyPasses == 2 && pass == 1) ? 5 - pi0 : pi0,
                    t8 = 8 * (it & 127);
          if (!kIdle || it < kItems) poly_fir_item<(WFIX > 0)>(Gf, W, Pt, ntaps, A.poly_nmi0, A.poly_nn, pi, t8, part);
          if (pass < kPolyPasses - 1) {
            park[2 * tid] = make_float4(part[0], part[1], part[2], part[3]);
            park[2 * tid + 1] = make_float4(part[4], part[5], part[6], part[7]);
          }
        }
        __syncthreads();  // every item is done reading G: its planes take the 4 x kPolyTC partial sums
        float* red = Gf;
  #pragma unroll
        for (int pass = 0; pass < kPolyPasses; pass++) {
          const int it = pass * kPolyThreads + tid, pi0 = it >> 7, pi = (kPolyPasses == 2 && pass == 1) ? 5 - pi0 : pi0,
                    t8 = 8 * (it & 127);
          if (kIdle && it >= kItems) break;
          float4* r4 = reinterpret_cast<float4*>(red + pi * kPolyTC + t8);
          if (pass < kPolyPasses - 1) {
            r4[0] = park[2 * tid];
            r4[1] = park[2 * tid + 1];
          } else {
            r4[0] = make_float4(part[0], part[1], part[2], part[3]);
            r4[1] = make_float4(part[4], part[5], part[6], part[7]);
          }
        }
      }
      __syncthreads();
      {
        const float* red = Gf;
  #pragma unroll
        for (int h = 0; h < kPolyTC / kPolyThreads; h++) {
          // the item's outputs: a sub-range of the tile under a split plan (512- and 1024-thread CTAs), else the tile
          const int t = tid + h * kPolyThreads, k = (THREADS >= 512 ? T.ot0 : T.t0) + t;
          if (k < (THREADS >= 512 ? T.ote : T.te))
            A.out[T.row + k] = (red[t] + red[kPolyTC + t]) + (red[2 * kPolyTC + t] + red[3 * kPolyTC + t]);
        }
        if (T.tail)
          poly_fused_tail(sm.ti, red, nullptr, tid, kPolyThreads, A.out, A.tail_win, A.tail_seed, 0, kPolyThreads);
      }
    }
    PTL_MARK(5);
    __syncthreads();  // G and the tile record are reused by the next work item
    PTL_MARK(6);
    PTL_ACC();
  }
  (void)lane; (void)warp;
}

static int poly_w(int ntaps) { return ntaps <= kPolyWFixTaps ? kPolyWFix : poly_plane_words(ntaps); }

template <int THREADS>
static size_t poly_smem_bytes(int ntaps, bool two_word, bool cluster = false) {
  (void)cluster;
  const size_t W = (size_t)poly_w(ntaps);
  return sizeof(PolySmem<THREADS>) + (two_word ? 2 : 1) * kPolyD * W * sizeof(int) +
         (size_t)poly_tab_floats(ntaps, kPolyMaxNear) * sizeof(float);
}

size_t ism_poly_smem_bytes(int ntaps, bool two_word) { return poly_smem_bytes<512>(ntaps, two_word); }

// cudaFuncSetAttribute is a driver call per launch otherwise (small calls are latency-bound): set the kernel's
// dynamic shared-memory limit (and the non-portable cluster size) once per device, to the most any call uses.
// The cache is per kernel INSTANTIATION (template parameters), not per function type: every variant of
// ism_poly_kernel has the same signature, and a cache keyed on the type set only the first one launched.
template <int THREADS, int WFIX, bool CL>
static cudaError_t ensure_attrs() {
  static unsigned long long done = 0;  // bit per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev >= 64) return e;
  if (__atomic_load_n(&done, __ATOMIC_ACQUIRE) & (1ull << dev)) return cudaSuccess;
  auto* kernel = ism_poly_kernel<THREADS, WFIX, CL>;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess && CL) e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) __atomic_fetch_or(&done, 1ull << dev, __ATOMIC_RELEASE);
  return e;
}

template <int THREADS, int WFIX>
static cudaError_t launch_poly_w(const IsmArgs& A, long long n_work, int* counter, size_t smem, int num_sms,
                                 cudaStream_t stream) {
  cudaError_t e = ensure_attrs<THREADS, WFIX, false>();
  if (e != cudaSuccess) return e;
  const long long slots = (long long)PolyCfg<THREADS>::kCtasPerSm * num_sms;
  const int grid = (int)(n_work < slots ? n_work : slots);
  ism_poly_kernel<THREADS, WFIX, false><<<grid, THREADS, smem, stream>>>(A, n_work, counter);
  return cudaGetLastError();
}
template <int THREADS>
static cudaError_t launch_poly(const IsmArgs& A, long long n_work, int* counter, size_t smem, int num_sms,
                               cudaStream_t stream) {
  return A.poly_ntaps <= kPolyWFixTaps ? launch_poly_w<THREADS, kPolyWFix>(A, n_work, counter, smem, num_sms, stream)
                                       : launch_poly_w<THREADS, 0>(A, n_work, counter, smem, num_sms, stream);
}

template <int THREADS, int WFIX>
static cudaError_t launch_poly_cluster(const IsmArgs& A, long long n_work, long long n_clusters, int S, size_t smem,
                                       cudaStream_t stream) {
  cudaError_t e = ensure_attrs<THREADS, WFIX, true>();
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_clusters * S), 1, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)S;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ism_poly_kernel<THREADS, WFIX, true>, A, n_work, (int*)nullptr);
}

// Clusters of S CTAs of THREADS threads with `smem` bytes each that the GPU holds at once (GPCs hold whole
// clusters); cached per device, shape and shared-memory size; 0 if the query fails.
template <int THREADS, int WFIX>
static int poly_max_clusters(int S, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<long long, int>> cache;  // key: (device, S, smem)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  const long long key = ((long long)dev << 40) | ((long long)S << 32) | (long long)smem;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& kv : cache)
      if (kv.first == key) return kv.second;
  }
  int n = 0;
  if (ensure_attrs<THREADS, WFIX, true>() == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)S, 1, 1);
    cfg.blockDim = dim3(THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, ism_poly_kernel<THREADS, WFIX, true>, &cfg) != cudaSuccess) {
      (void)cudaGetLastError();
      n = 0;
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  cache.emplace_back(key, n);
  return n;
}

static int poly_max_clusters_for(int threads, int S, int ntaps, bool two_word) {
  if (threads == 1024) {
    const size_t smem = poly_smem_bytes<1024>(ntaps, two_word, true);
    return ntaps <= kPolyWFixTaps ? poly_max_clusters<1024, kPolyWFix>(S, smem) : poly_max_clusters<1024, 0>(S, smem);
  }
  const size_t smem = poly_smem_bytes<512>(ntaps, two_word, true);
  return ntaps <= kPolyWFixTaps ? poly_max_clusters<512, kPolyWFix>(S, smem) : poly_max_clusters<512, 0>(S, smem);
}

// Shape of a call's items: 0 = persistent CTAs; else clusters of S CTAs of `threads` threads, one item per
// cluster.  Small calls (fewer than 2 items per SM): S = 4..16 such that the call has about 2 CTAs per SM, and
// 1024-thread CTAs (one per SM: all 32 warps hide the image walk's latencies; config 1: 18.7 vs 20.6 us per call)
// when the GPU holds all its clusters at that size in one wave (GPCs hold whole clusters), else 512-thread CTAs.
// split > 0 forces S (512 threads), split < 0 persistent CTAs.  GPURIR_POLY_CL_THREADS=512: always 512 (A/B).
int ism_poly_cluster_size(long long n_work, int num_sms, int split, int ntaps, bool two_word, int* threads) {
  static const bool only512 = [] {
    const char* e = getenv("GPURIR_POLY_CL_THREADS");
    return e && atoi(e) == 512;
  }();
  if (threads) *threads = 512;
  if (split > 0) return split;
  // cluster items only for the smallest calls: from ~32 items persistent CTAs (one per item, heavy tiles' output ranges
  // split over the idle SMs) are faster, while clusters of 4-8 CTAs per tile pay their exchange and run in several
  // waves (graph-timed, tools/mid_calls.py: 8 receivers of config 3 (i) 19.9 vs 26.3 us, 12: 30.0 vs 25.8 us)
  static const long long cl_max = [] {  // GPURIR_POLY_CL_MAX: A/B of the threshold
    const char* e = getenv("GPURIR_POLY_CL_MAX");
    return e ? atoll(e) : (long long)kPolyClusterMaxItems;
  }();
  if (split < 0 || n_work >= 2LL * num_sms || n_work > cl_max) return 0;
  int S = 4;
  while (S < 16 && n_work * S < 2LL * num_sms) S *= 2;
  // items whose output ranges the planner may split (poly_plan_subs) get clusters of 8: sub-ranges add the
  // clusters; measured best at 8 with 1024-thread CTAs (config 2 at T60 = 2 s: 18.6 vs 20.7 us per call at 16)
  if (n_work <= kPolyMaxItems) S = 8;
  static const int force_s = [] {
    const char* e = getenv("GPURIR_POLY_CL_S");  // A/B of the cluster size of small calls
    const int x = e ? atoi(e) : 0;
    return (x == 4 || x == 8 || x == 16) ? x : 0;
  }();
  if (force_s) S = force_s;
  if (!only512 && n_work <= poly_max_clusters_for(1024, S, ntaps, two_word) && threads) *threads = 1024;
  return S;
}

// L2 exchange scratch of a cluster-item launch: a slab of 2 kPolyD planes per CTA, for at most max(items x S,
// 2 x SMs) CTAs (output sub-ranges add clusters only up to one wave)
size_t ism_poly_slab_words(long long n_work, int S, int ntaps, int num_sms) {
  if (S <= 0) return 0;
  const size_t Ws = (size_t)((kPolyTC + ntaps - 1 + 31) & ~31);
  const long long ctas = std::max(n_work * S, 2LL * num_sms + S);
  return (size_t)ctas * 2 * kPolyD * Ws;
}

// Output sub-ranges of a small single-room call's items (IsmArgs::poly_first): item wi is tile nTiles - 1 - wi / M
// of RIR wi % M (end-aligned 1024-sample tiles); its images lie in the shell of delays (t0 - H, te + H), about
// (te + H)^3 - (t0 - H)^3 of them.  Starting from one cluster per item, the full tile with the most images per
// cluster is split in two (then four) while the GPU holds all clusters in one wave (cmax) — the last tile only while
// its last part still holds the fused tail's envelope window.  Returns the cluster count.
static long long poly_plan_subs(IsmArgs& B, long long n_work, long long cmax) {
  const double H = 0.5 * B.poly_ntaps;
  std::vector<double> w((size_t)n_work);
  std::vector<int> ns((size_t)n_work, 1);
  std::vector<char> full((size_t)n_work), last((size_t)n_work);
  for (long long wi = 0; wi < n_work; wi++) {
    const int tile = B.nTiles - 1 - (int)(wi / B.M);
    const long long te = B.nISM - (long long)(B.nTiles - 1 - tile) * kPolyTC, t0 = std::max(0LL, te - kPolyTC);
    const double lo = std::max(0.0, (double)t0 - H), hi = (double)te + H;
    w[(size_t)wi] = hi * hi * hi - lo * lo * lo;
    full[(size_t)wi] = te - t0 == kPolyTC;
    last[(size_t)wi] = tile == B.nTiles - 1;
  }
  long long total = n_work;
  for (;;) {
    long long best = -1;
    double worst = 0.0;
    for (long long wi = 0; wi < n_work; wi++) {
      const int k = ns[(size_t)wi];
      if (!full[(size_t)wi] || k >= 4) continue;
      if (last[(size_t)wi] && B.poly_tail && kPolyTC / (2 * k) < B.tail_win) continue;
      if (w[(size_t)wi] / k > worst) { worst = w[(size_t)wi] / k; best = wi; }
    }
    if (best < 0 || total + ns[(size_t)best] > cmax) break;
    total += ns[(size_t)best];
    ns[(size_t)best] *= 2;
  }
  // a partial (first) tile holds few images but still all its outputs on one cluster, whose exchange and filter then
  // finish last (config 1: 704 outputs): split it in two when there is room
  for (long long wi = 0; wi < n_work; wi++) {
    const int tile = B.nTiles - 1 - (int)(wi / B.M);
    const long long te = B.nISM - (long long)(B.nTiles - 1 - tile) * kPolyTC, t0 = std::max(0LL, te - kPolyTC);
    if (full[(size_t)wi] || ns[(size_t)wi] != 1 || te - t0 <= kPolyTC / 2 || total + 1 > cmax) continue;
    if (last[(size_t)wi] && B.poly_tail && (((te - t0 + 1) / 2 + 127) & ~127) < B.tail_win) continue;
    ns[(size_t)wi] = 2;
    total += 1;
  }
  if (total > kPolyMaxSubItems) return n_work;  // (cannot happen: cmax is at most one wave) no plan
  int first = 0;
  for (long long wi = 0; wi < n_work; wi++) {
    B.poly_first[wi] = (unsigned short)first;
    const int k = ns[(size_t)wi], lg = k == 4 ? 2 : k == 2 ? 1 : 0;
    for (int sub = 0; sub < k; sub++) B.poly_cmap[first + sub] = (unsigned short)(wi | sub << 10 | lg << 12);
    first += k;
  }
  B.poly_first[n_work] = (unsigned short)first;
  B.poly_nitems = (int)n_work;
  return total;
}

cudaError_t launch_ism_poly(const IsmArgs& A, long long n_work, int* counter, int num_sms, int split,
                            cudaStream_t stream) {
  const bool two_word = A.poly_gbz != 0;  // some tile starts in the two-word format
  IsmArgs B = A;
  int cl_threads = 512;
  const int S = ism_poly_cluster_size(n_work, num_sms, split, A.poly_ntaps, two_word, &cl_threads);
  if (S > 0) {  // cluster items: no redo, so the fine plane only for two-word tiles
    if (S != 4 && S != 8 && S != 16) return cudaErrorInvalidValue;
    if (!A.poly_slab || A.poly_slab_w < kPolyTC + A.poly_ntaps - 1) return cudaErrorInvalidValue;
    B.poly_gb = two_word;
    B.poly_nitems = 0;
    long long n_clusters = n_work;
    if (split == 0 && !A.jobs && n_work <= kPolyMaxItems) {  // heavy tiles' output ranges over more clusters
      const long long cmax = poly_max_clusters_for(cl_threads, S, A.poly_ntaps, two_word);
      const long long cap = std::min(cmax, (2LL * num_sms + S) / S);  // the exchange scratch is sized for this
      if (cap > n_work) n_clusters = poly_plan_subs(B, n_work, cap);
    }
    if (cl_threads == 1024) {
      const size_t smem = poly_smem_bytes<1024>(A.poly_ntaps, two_word, true);
      return A.poly_ntaps <= kPolyWFixTaps ? launch_poly_cluster<1024, kPolyWFix>(B, n_work, n_clusters, S, smem, stream)
                                           : launch_poly_cluster<1024, 0>(B, n_work, n_clusters, S, smem, stream);
    }
    const size_t smem = poly_smem_bytes<512>(A.poly_ntaps, two_word, true);
    return A.poly_ntaps <= kPolyWFixTaps ? launch_poly_cluster<512, kPolyWFix>(B, n_work, n_clusters, S, smem, stream)
                                         : launch_poly_cluster<512, 0>(B, n_work, n_clusters, S, smem, stream);
  }
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  const size_t s256 = poly_smem_bytes<256>(A.poly_ntaps, false);
  // 256-thread CTAs (4 per SM) from 7 items per SM: graph-timed on config 3 (i) (tools/mid_calls.py --large), 7.8 items
  // per SM 105 vs 109 us, 15.6: 193 vs 208 us, but 5.2: 86 vs 79 us (fewer, wider CTAs keep the heavy tiles moving)
  static const long long min256 = [] {  // GPURIR_POLY_MIN256: A/B of the threshold (items per SM)
    const char* e = getenv("GPURIR_POLY_MIN256");
    return e ? atoll(e) : 7LL;
  }();
  if (!two_word && 4 * s256 <= 224 * 1024 && n_work >= min256 * num_sms) {
    B.poly_gb = 0;
    return launch_poly<256>(B, n_work, counter, s256, num_sms, stream);
  }
  // at most one item per SM: one 1024-thread CTA per item (twice the warps of a 512-thread CTA on each tile; the fine
  // plane always fits), the same bits as every other shape
  static const bool no1024 = getenv("GPURIR_POLY_NO1024") != nullptr;  // A/B switch
  static const bool nosub = getenv("GPURIR_POLY_NOSUB") != nullptr;     // A/B switch: no output-range splits
  if (n_work <= num_sms && !no1024) {
    B.poly_gb = 1;
    // heavy tiles' output ranges split over the idle SMs (as for cluster items; each part its own CTA and queue
    // entry, enumerating only its thin shell of images, with the whole tile's fixed-point format: the same bits)
    long long n_entries = n_work;
    B.poly_nitems = 0;
    if (split == 0 && !A.jobs && n_work <= kPolyMaxItems && !nosub) n_entries = poly_plan_subs(B, n_work, num_sms);
    return launch_poly<1024>(B, n_entries, counter, poly_smem_bytes<1024>(A.poly_ntaps, true), num_sms, stream);
  }
  // 512-thread CTAs carry the fine plane whenever two of them still fit an SM with it (the guard's redo)
  const size_t s1 = poly_smem_bytes<512>(A.poly_ntaps, false), s2 = poly_smem_bytes<512>(A.poly_ntaps, true);
  B.poly_gb = two_word || 2 * (s2 + 1024) <= 228 * 1024;
  // up to two items per SM: the heavy tiles' output ranges split over the free CTA slots, as above
  long long n_entries = n_work;
  B.poly_nitems = 0;
  if (split == 0 && !A.jobs && n_work <= 2LL * num_sms && n_work <= kPolyMaxItems && !nosub)
    n_entries = poly_plan_subs(B, n_work, 2LL * num_sms);
  return launch_poly<512>(B, n_entries, counter, B.poly_gb ? s2 : s1, num_sms, stream);
}

}  // namespace gpurir

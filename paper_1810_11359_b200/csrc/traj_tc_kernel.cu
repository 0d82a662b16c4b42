// traj_tc_kernel.cu — NEXT row f1 of SURVEY.md §8(f) on the 5th-generation tensor cores (tcgen05): a moving
// source recorded by a microphone array (§3.4), the same linear filter as traj_kernel.cu
// (reading R7 = SPEC S:414):
//
//   out[m][t] = sum_j sig[j] rir[p(j)][m][t - j],   p(j) = min(j / floor(n_sig / n_points), n_points - 1).
//
// As a GEMM.  Segment p covers inputs [j_p, e_p); pad it to U = 4 ceil((e_p - j') / 4) + 1 samples from the
// 32-aligned j' = 32 floor(j_p / 32) (zeros outside [j_p, e_p)).  For a block of 128 outputs t = t0 + i
// (t0 = 128 a) its contribution is
//
//   y[t0 + i] = sum_u s'[u] r[t0 + i - j' - u] = sum_k A[i][k] B[k],   k = i - u + U - 1 in [0, 127 + U),
//   A[i][k] = s'[i + U - 1 - k]  (a banded Toeplitz matrix of the SIGNAL, the same for every block and mic),
//   B[k]    = r_{p,m}[base_a + k],  base_a = t0 - j' - (U - 1)  (a window of the RIR, zero outside [0, L)).
//
// So one tile D[128 x N] = out[m][128 a + i] for N (block a, mic m) columns is the sum over the segments and
// 32-wide K chunks of A_chunk[128 x 32] B_chunk[32 x N]: M = 128, N = 256, K = 32 per chunk, with the A chunk
// shared by all columns.  fp32 accuracy from the tf32 tensor cores by the 3xTF32 split: x = hi + lo with
// hi = x with its 13 low mantissa bits cleared (exact in tf32) and lo = x - hi (exact in fp32, ~2^-11 x); each
// chunk accumulates A_hi B_hi + A_hi B_lo + A_lo B_hi in fp32 (TMEM) — the dropped A_lo B_lo and the tf32
// truncation of lo are ~2^-22 of each product (tolerance R8: 2e-5 of the output peak).
//
// One CTA = one tile (or one K-split share of it: the per-split partial tiles are summed in split order by
// traj_reduce_kernel, so the result is deterministic).  Warp 0 allocates TMEM and one elected thread issues the
// tcgen05.mma (kind::tf32, cta_group::1; 12 per chunk: 3 products x 4 K-steps of 8); warps 1..11 produce: for
// chunk q they load the signal (A) and RIR windows (B, 16-B loads) into registers, wait until stage q % 2 is
// free (tcgen05.commit of chunk q - 2 arrives on its mbarrier), split hi/lo and store both into the stage in
// the UMMA canonical K-major layout (consecutive 16-B rows: conflict-free stores), fence.proxy.async, and arrive
// on the stage's "full" mbarrier.  After the last chunk the MMA thread commits to the "done" mbarrier; warps
// 4..7 read D from TMEM (32x32b loads: warp q holds rows 32 q .. 32 q + 31) and store it coalesced.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <vector>

#include <cuda.h>

#include "kernels.h"
#include "tc_common.cuh"

namespace gpurir {

using namespace tc;

constexpr int kTcM = 128;                            // outputs per block (rows of D, TMEM lanes)
constexpr int kTcN = 256;                            // (block, mic) columns per tile (TMEM columns)
constexpr int kTcStages = 2;
constexpr int kTcThreads = 384;                      // warp 0: TMEM + MMA issue; warp 1: TMA; warps 2..11: producers
constexpr int kTcProd = kTcThreads - 64;
constexpr int kTcAItems = kTcM * 8;                  // 16-B groups of an A chunk (128 rows x 8)
constexpr int kTcBItems = kTcN * 8;                  // 16-B groups of a B chunk (256 columns x 8)
constexpr int kTcABytes = kTcM * 32 * 4;             // 16 KB
constexpr int kTcBBytes = kTcN * 32 * 4;             // 32 KB
constexpr int kTcStageBytes = 2 * kTcABytes + kTcBBytes;  // A hi, A lo, B lo: 64 KB
constexpr int kTcRing = 3;                           // slots of raw B (the MMA's B hi), one chunk ahead of the stages
constexpr int kTcMaxTiles = 1024;                    // tiles of one call (the CTA table is a kernel parameter)

struct TrajTcArgs {
  const float* sig;
  long long n_sig;
  const float* rirs;
  int n_points, n_mics;
  long long L;
  long long n_out;
  long long seglen;
  int nA;       // blocks of 128 outputs
  int n_cols;   // nA * n_mics  (column c = a * n_mics + m)
  float* out;   // [n_mics][n_out]
  float* part;  // per CTA of a split tile: its partial tile [kTcN columns][kTcM rows]
  int n_tiles;
  int tma_rows;  // rows (mics) per TMA box of B: 32 when n_mics % 32 == 0, else 8
  unsigned short cta_first[kTcMaxTiles + 1];  // CTAs of tile t: [cta_first[t], cta_first[t + 1]) (K shares)
};

struct TcSeg {
  long long jp, ep, j0;  // inputs [jp, ep); 32-aligned start j0 <= jp
  long long U;           // padded length, U - 1 a multiple of 4
  int nC;                // K chunks: ceil((127 + U) / 32)
};

__host__ __device__ __forceinline__ TcSeg tc_seg(const TrajTcArgs& P, int p) {
  TcSeg s;
  s.jp = (long long)p * P.seglen;
  s.ep = p == P.n_points - 1 ? P.n_sig : s.jp + P.seglen;
  s.j0 = s.jp & ~31LL;
  s.U = 4 * ((s.ep - s.j0 + 3) / 4) + 1;
  s.nC = (int)((127 + s.U + 31) / 32);
  return s;
}

// Chunks of segment p that touch the tile's blocks [a_lo, a_hi]: k in [-base_{a_hi}, L - base_{a_lo}) n [0, K)
__host__ __device__ __forceinline__ void tc_chunks(const TrajTcArgs& P, const TcSeg& s, int a_lo, int a_hi, int& c0, int& c1) {
  const long long off = -s.j0 - (s.U - 1);
  const long long klo = -(128LL * a_hi + off), khi = P.L - (128LL * a_lo + off);  // [klo, khi)
  long long lo = klo > 0 ? klo / 32 : 0;
  long long hi = khi <= 0 ? -1 : (khi - 1) / 32;
  if (hi > s.nC - 1) hi = s.nC - 1;
  c0 = (int)lo;
  c1 = (int)hi;
}

// Segments that reach the tile's outputs [128 a_lo, 128 (a_hi + 1)): y_p covers t in [j_p, e_p + L - 2]
__host__ __device__ __forceinline__ void tc_segs(const TrajTcArgs& P, int a_lo, int a_hi, int& p0, int& p1) {
  const long long tlo = 128LL * a_lo, thi = 128LL * (a_hi + 1) - 1;
  long long lo = (tlo - P.L + 2) / P.seglen - 1;  // a safe lower bound (one below), refined below
  if (lo < 0) lo = 0;
  while (lo < P.n_points - 1 && tc_seg(P, (int)lo).ep + P.L - 2 < tlo) lo++;
  long long hi = thi / P.seglen;
  if (hi > P.n_points - 1) hi = P.n_points - 1;
  p0 = (int)lo;
  p1 = (int)hi;
}

// Walks this CTA's share [q_begin, q_end) of the tile's chunk list (segments ascending, chunks ascending).
struct TcWalk {
  int p, p1, c, c1;
  TcSeg s;
  int a_lo, a_hi;
  __host__ __device__ bool next_seg(const TrajTcArgs& P) {
    for (; p <= p1; p++) {
      s = tc_seg(P, p);
      tc_chunks(P, s, a_lo, a_hi, c, c1);
      if (c <= c1) return true;
    }
    return false;
  }
  // position on chunk index q (counting from the tile's first chunk); false if the list is shorter
  __host__ __device__ bool seek(const TrajTcArgs& P, int p0, long long q) {
    p = p0;
    for (;;) {
      if (!next_seg(P)) return false;
      const int n = c1 - c + 1;
      if (q < n) { c += (int)q; return true; }
      q -= n;
      p++;
    }
  }
  __host__ __device__ bool advance(const TrajTcArgs& P) {
    if (++c <= c1) return true;
    p++;
    return next_seg(P);
  }
};

// The tile's chunk count (the same walk on the host, to balance the K shares, and in every CTA)
__host__ __device__ inline long long tc_tile_chunks(const TrajTcArgs& P, int tile, int& a_lo, int& a_hi, int& p0,
                                                   int& p1) {
  const int col0 = tile * kTcN;
  a_lo = col0 / P.n_mics;
  a_hi = (col0 + kTcN - 1) / P.n_mics;
  if (a_hi > P.nA - 1) a_hi = P.nA - 1;
  tc_segs(P, a_lo, a_hi, p0, p1);
  long long Q = 0;
  TcWalk w;
  w.p = p0; w.p1 = p1; w.a_lo = a_lo; w.a_hi = a_hi;
  while (w.next_seg(P)) { Q += w.c1 - w.c + 1; w.p++; }
  return Q;
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// Shared-memory map of the kernel (dynamic; the 128-B swizzle is a function of the address bits, so the base must
// be 1024-B aligned — it is, with no static shared memory — and the kernel traps otherwise): kTcStages stages of
// {A hi, A lo, B lo}, kTcRing slots of raw B (fp32 RIR windows: the tensor core truncates them to tf32, i.e. they
// are B hi; the TMA fills them a chunk ahead of the stages), per stage the signal window of the chunk's A, and
// the mbarriers.
constexpr int kTcZWin = kTcM + 32;                 // z values one chunk's A reads: z[32 c - 127 .. 32 c + 31]
constexpr int kTcSmemBytes = kTcStages * kTcStageBytes + kTcRing * kTcBBytes + kTcStages * kTcZWin * 4 + 256;

template <bool kTma>
__global__ void __launch_bounds__(kTcThreads, 1) traj_tc_kernel(const __grid_constant__ TrajTcArgs P,
                                                                 const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ring = smem + kTcStages * kTcStageBytes;                                 // [kTcRing] raw B
  float* zwin = reinterpret_cast<float*>(ring + kTcRing * kTcBBytes);                    // [kTcStages][kTcZWin]
  uint64_t* bars = reinterpret_cast<uint64_t*>(zwin + kTcStages * kTcZWin);
  uint64_t* full_bar = bars;                          // producers' arrivals (A, B lo built; raw B landed)
  uint64_t* empty_bar = bars + kTcStages;             // tcgen05.commit: the stage's MMAs are done
  uint64_t* raw_bar = bars + 2 * kTcStages;           // TMA bytes of a ring slot
  uint64_t* ring_bar = bars + 2 * kTcStages + kTcRing;  // tcgen05.commit: the ring slot's MMAs are done
  uint64_t* done_bar = bars + 2 * kTcStages + 2 * kTcRing;
  uint32_t* tmem_base = reinterpret_cast<uint32_t*>(done_bar + 1);
  if ((smem_u32(smem) & 1023) != 0) __trap();  // the swizzled operands need a 1024-B aligned base
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // this CTA's tile (the last t with cta_first[t] <= blockIdx.x) and its K share of the tile's chunk list
  int tile = 0;
  {
    int lo = 0, hi = P.n_tiles - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)P.cta_first[mid] <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
    }
    tile = lo;
  }
  const int split = (int)blockIdx.x - (int)P.cta_first[tile];
  const int nsplit = (int)P.cta_first[tile + 1] - (int)P.cta_first[tile];
  const int col0 = tile * kTcN;
  int a_lo, a_hi, p0, p1;
  const long long Q = tc_tile_chunks(P, tile, a_lo, a_hi, p0, p1);
  const long long q_begin = Q * split / nsplit, q_end = Q * (split + 1) / nsplit;
  const int nq = (int)(q_end - q_begin);

  if (warp == 0) tmem_alloc(tmem_base, kTcN);
  if (tid == 32) {
    for (int s = 0; s < kTcStages; s++) {
      mbar_init(&full_bar[s], kTcProd / 32);
      mbar_init(&empty_bar[s], 1);
    }
    for (int r = 0; r < kTcRing; r++) {
      mbar_init(&raw_bar[r], 1);
      mbar_init(&ring_bar[r], 1);
    }
    mbar_init(done_bar, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_base;

  if (warp == 0) {
    // ---- MMA issue (one thread): 3 products x 4 K steps of 8 per chunk ----
    if (lane == 0 && nq > 0) {
      const uint32_t idesc = idesc_tf32(kTcM, kTcN);
      for (int q = 0; q < nq; q++) {
        const int st = q % kTcStages;
        mbar_wait(&full_bar[st], (uint32_t)((q / kTcStages) & 1));
        tc_fence_after();
        const unsigned char* base = smem + (size_t)st * kTcStageBytes;
        const uint64_t dah = smem_desc_sw128(base), dal = smem_desc_sw128(base + kTcABytes);
        const uint64_t dbh = smem_desc_sw128(ring + (size_t)(q % kTcRing) * kTcBBytes);
        const uint64_t dbl = smem_desc_sw128(base + 2 * kTcABytes);
#pragma unroll
        for (int k = 0; k < 4; k++) {  // +32 B per K step: descriptor + 2 (16-B units)
          mma_tf32(tmem, dah + 2 * k, dbh + 2 * k, idesc, q > 0 || k > 0);
          mma_tf32(tmem, dah + 2 * k, dbl + 2 * k, idesc, true);
          mma_tf32(tmem, dal + 2 * k, dbh + 2 * k, idesc, true);
        }
        mma_commit(&empty_bar[st]);            // the stage is free once these MMAs have read it
        mma_commit(&ring_bar[q % kTcRing]);    // and so is the ring slot
      }
      mma_commit(done_bar);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---- TMA issue (one thread): the chunk's B = 32 boxes of 8 (block, mic) rows x 32 samples (1 KB each) ----
    if (kTma && lane == 0 && nq > 0) {
      TcWalk w;
      w.p1 = p1; w.a_lo = a_lo; w.a_hi = a_hi;
      bool ok = w.seek(P, p0, q_begin);
      for (int q = 0; q < nq && ok; q++) {
        const int rs = q % kTcRing;
        if (q >= kTcRing) mbar_wait(&ring_bar[rs], (uint32_t)(((q / kTcRing) - 1) & 1));
        // boxes of P.tma_rows (8 or 32) consecutive mics of one block (n_mics is a multiple of tma_rows)
        const int ng = min(kTcN, P.n_cols - col0) / P.tma_rows;
        mbar_arrive_expect_tx(&raw_bar[rs], (uint32_t)(ng * P.tma_rows * 128));
        unsigned char* braw = ring + (size_t)rs * kTcBBytes;
        const int xb = (int)(-w.s.j0 - (w.s.U - 1) + 32LL * w.c);
        for (int g = 0; g < ng; g++) {
          const int col = col0 + P.tma_rows * g, a = col / P.n_mics, m0 = col - a * P.n_mics;
          tma_load_2d(braw + 128 * P.tma_rows * g, &tmap, 128 * a + xb, w.p * P.n_mics + m0, &raw_bar[rs]);
        }
        ok = w.advance(P);
      }
    }
  } else {
    // ---- producers (warps 2..11): per chunk the signal window, A hi / lo, B lo (and B raw without TMA) ----
    const int pt = tid - 64;
    constexpr int kNP = kTcProd;
    TcWalk w;
    w.p1 = p1; w.a_lo = a_lo; w.a_hi = a_hi;
    bool ok = nq > 0 && w.seek(P, p0, q_begin);
    // B without TMA: this thread's groups (column, K quarter) and their fp32 values, one chunk ahead
    constexpr int kBPer = (kTcBItems + kNP - 1) / kNP;
    int b_off[kBPer];
    long long b_row[kBPer];
    float4 bv[kBPer];
    if (!kTma) {
#pragma unroll
      for (int r = 0; r < kBPer; r++) {
        const int it = pt + r * kNP, n = it >> 3, kq = it & 7, col = col0 + n;
        if (it < kTcBItems && col < P.n_cols) {
          const int a = col / P.n_mics, m = col - a * P.n_mics;
          b_off[r] = 128 * a + 4 * kq;
          b_row[r] = (long long)m * P.L;
        } else {
          b_off[r] = INT_MIN;
          b_row[r] = 0;
        }
      }
    }
    auto zval = [&]() {  // z[x] = s'[U - 1 - x] for this thread's window slot x = 32 c - 127 + pt
      const TcSeg& s = w.s;
      const long long x = 32LL * w.c - (kTcM - 1) + pt, g = s.j0 + s.U - 1 - x;
      return (pt < kTcZWin && x >= 0 && x < s.U && g >= s.jp && g < s.ep) ? __ldg(P.sig + g) : 0.f;
    };
    auto bload = [&]() {
      const TcSeg& s = w.s;
      const long long xb = -s.j0 - (s.U - 1) + 32LL * w.c;
      const float* bank = P.rirs + (long long)w.p * P.n_mics * P.L;
#pragma unroll
      for (int r = 0; r < kBPer; r++) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (b_off[r] != INT_MIN) {  // base_a, L multiples of 4: the 4 samples are all in or all out
          const long long x0 = xb + b_off[r];
          if (x0 >= 0 && x0 < P.L) v = __ldg(reinterpret_cast<const float4*>(bank + b_row[r] + x0));
        }
        bv[r] = v;
      }
    };
    float zr = 0.f;
    if (ok) {
      zr = zval();
      if (!kTma) bload();
    }
    for (int q = 0; q < nq && ok; q++) {
      const int st = q % kTcStages;
      if (q >= kTcStages) mbar_wait(&empty_bar[st], (uint32_t)(((q / kTcStages) - 1) & 1));
      unsigned char* base = smem + (size_t)st * kTcStageBytes;
      float* zw = zwin + st * kTcZWin;
      if (pt < kTcZWin) zw[pt] = zr;
      if (!kTma) {  // B raw (the MMA truncates it to tf32) and B lo from the registers
#pragma unroll
        for (int r = 0; r < kBPer; r++) {
          const int it = pt + r * kNP;
          if (it < kTcBItems) {
            const float4 v = bv[r];
            const int off = sw128_off(it >> 3, 4 * (it & 7));
            *reinterpret_cast<float4*>(ring + (size_t)(q % kTcRing) * kTcBBytes + off) = v;  // free: MMA q - 3 is done
            *reinterpret_cast<float4*>(base + 2 * kTcABytes + off) =
                make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kNP) : "memory");  // the window is complete
      // A[i][32 c + 4 kq + e] = z[32 c + 4 kq + e - i] = zw[4 kq + e - i + 127]
      for (int it = pt; it < kTcAItems; it += kNP) {
        const int i = it >> 3, kq = it & 7;
        const float* zp = zw + 4 * kq - i + (kTcM - 1);
        const float4 v = make_float4(zp[0], zp[1], zp[2], zp[3]);
        const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        const int off = sw128_off(i, 4 * kq);
        *reinterpret_cast<float4*>(base + off) = h;
        *reinterpret_cast<float4*>(base + kTcABytes + off) = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
      }
      // the next chunk's loads go out before this chunk's B lo (they overlap the TMA wait and the smem work)
      ok = w.advance(P);
      const bool more = q + 1 < nq && ok;
      if (more) {
        zr = zval();
        if (!kTma) bload();
      }
      if (kTma) {
        mbar_wait(&raw_bar[q % kTcRing], (uint32_t)((q / kTcRing) & 1));  // the TMA boxes of B have landed
        const unsigned char* braw = ring + (size_t)(q % kTcRing) * kTcBBytes;
        for (int it = pt; it < kTcBItems; it += kNP) {
          const int off = sw128_off(it >> 3, 4 * (it & 7));
          const float4 v = *reinterpret_cast<const float4*>(braw + off);
          *reinterpret_cast<float4*>(base + 2 * kTcABytes + off) =
              make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y), v.z - tf32_hi(v.z), v.w - tf32_hi(v.w));
        }
      }
      fence_proxy_async();  // this thread's stores are visible to the tensor cores
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[st]);
    }
  }

  // ---- epilogue: warps 4..7 read D (rows 32 (warp - 4) ...) and store (block a, mic m) columns ----
  if (warp >= 4 && warp < 8) {
    const int q4 = warp - 4, row = 32 * q4 + lane;
    if (nq > 0) {
      mbar_wait(done_bar, 0);
      tc_fence_after();
    }
    float* part = nsplit > 1 ? P.part + (size_t)blockIdx.x * kTcN * kTcM : nullptr;
    for (int c0 = 0; c0 < kTcN; c0 += 16) {
      float v[16];
      if (nq > 0) {
        tmem_ld16(tmem + ((uint32_t)(32 * q4) << 16) + (uint32_t)c0, v);
      } else {
#pragma unroll
        for (int j = 0; j < 16; j++) v[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; j++) {
        if (part) {  // partial tile [column][row], summed by traj_reduce_kernel
          part[(size_t)(c0 + j) * kTcM + row] = v[j];
          continue;
        }
        const int col = col0 + c0 + j;
        if (col < P.n_cols) {
          const int a = col / P.n_mics, m = col - a * P.n_mics;
          const long long t = 128LL * a + row;
          if (t < P.n_out) P.out[(long long)m * P.n_out + t] = v[j];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTcN);
}

// Tiles split into K shares: out = the sum of the tile's partials in share order (deterministic).  One thread per
// element of a split tile ([kTcN columns][kTcM rows]); the shares' loads are all issued before the sum.
__global__ void traj_reduce_kernel(TrajTcArgs P) {
  const int tile = blockIdx.y, b0 = P.cta_first[tile], nb = (int)P.cta_first[tile + 1] - b0;
  if (nb <= 1) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // [column][row] element of the tile
  const int nn = e >> 7, row = e & 127;
  const int col = tile * kTcN + nn;
  if (col >= P.n_cols) return;
  const int a = col / P.n_mics, m = col - a * P.n_mics;
  const long long t = 128LL * a + row;
  if (t >= P.n_out) return;
  const float* src = P.part + (size_t)b0 * kTcN * kTcM + e;
  float acc = 0.f;
  for (int b = 0; b < nb; b += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) v[u] = b + u < nb ? __ldcg(src + (size_t)(b + u) * kTcN * kTcM) : 0.f;
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (b + u < nb) acc = (b + u == 0) ? v[u] : acc + v[u];
  }
  P.out[(long long)m * P.n_out + t] = acc;
}

bool traj_tc_supported(const float* rirs, long long L) {
  return (L % 4) == 0 && (reinterpret_cast<uintptr_t>(rirs) & 15) == 0;
}

// cuTensorMapEncodeTiled from the driver (no link-time libcuda dependency)
typedef CUresult (*TcEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                               const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TcEncodeFn tc_tensor_map_encoder() {
  static TcEncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<TcEncodeFn>(p);
  }();
  return fn;
}

static void traj_tc_args(TrajTcArgs& P, const float* sig, long long n_sig, const float* rirs, int n_points,
                         int n_mics, long long L) {
  P.sig = sig; P.n_sig = n_sig; P.rirs = rirs; P.n_points = n_points; P.n_mics = n_mics; P.L = L;
  P.n_out = n_sig + L - 1;
  P.seglen = n_sig / n_points;
  // counts in 64 bits first: a call whose tiles do not fit the CTA table (or int) runs the CUDA-core kernel
  const long long nA = (P.n_out + kTcM - 1) / kTcM, n_cols = nA * n_mics, n_tiles = (n_cols + kTcN - 1) / kTcN;
  const bool fits = n_tiles <= kTcMaxTiles;
  P.nA = fits ? (int)nA : 0;
  P.n_cols = fits ? (int)n_cols : 0;
  P.n_tiles = fits ? (int)n_tiles : kTcMaxTiles + 1;
}

// K shares per tile: about one CTA per SM in all, each with ~the same number of chunks (tiles at the ends of the
// output see few segments); force > 0 gives every tile min(force, chunks) shares (test hook).  Returns the CTA
// count (0: too many tiles for the CTA table — the CUDA-core kernel then runs).
static int traj_tc_plan(TrajTcArgs& P, int num_sms, int force) {
  if (P.n_tiles > kTcMaxTiles) return 0;
  std::vector<long long> Q((size_t)P.n_tiles);
  long long total = 0;
  for (int t = 0; t < P.n_tiles; t++) {
    int a_lo, a_hi, p0, p1;
    Q[(size_t)t] = tc_tile_chunks(P, t, a_lo, a_hi, p0, p1);
    total += Q[(size_t)t];
  }
  // shares k_t ~ Q_t num_sms / total, at least one per tile, at most num_sms CTAs in all (one wave): start from
  // the floor and hand the remaining CTAs to the tiles with the most chunks per share
  std::vector<long long> k((size_t)P.n_tiles);
  long long used = 0;
  for (int t = 0; t < P.n_tiles; t++) {
    k[(size_t)t] = force > 0 ? force : std::max(1LL, Q[(size_t)t] * num_sms / std::max(1LL, total));
    k[(size_t)t] = std::max(1LL, std::min(k[(size_t)t], std::max(1LL, Q[(size_t)t])));
    used += k[(size_t)t];
  }
  while (force <= 0 && used < num_sms) {
    int best = -1;
    double worst = 0.0;
    for (int t = 0; t < P.n_tiles; t++) {
      const double per = (double)Q[(size_t)t] / (double)k[(size_t)t];
      if (k[(size_t)t] < Q[(size_t)t] && per > worst) { worst = per; best = t; }
    }
    if (best < 0) break;
    k[(size_t)best]++;
    used++;
  }
  int n = 0;
  for (int t = 0; t < P.n_tiles; t++) {
    P.cta_first[t] = (unsigned short)n;
    n += (int)k[(size_t)t];
    if (n > 65535) return 0;
  }
  P.cta_first[P.n_tiles] = (unsigned short)n;
  return n;
}

size_t traj_tc_part_words(const float* sig, long long n_sig, const float* rirs, int n_points, int n_mics, long long L,
                          int num_sms, int force) {
  TrajTcArgs P;
  traj_tc_args(P, sig, n_sig, rirs, n_points, n_mics, L);
  const int n = traj_tc_plan(P, num_sms, force);
  return n > 0 ? (size_t)n * kTcN * kTcM : 0;
}

cudaError_t launch_traj_tc(const float* sig, long long n_sig, const float* rirs, int n_points, int n_mics, long long L,
                           float* out, float* partial, int num_sms, int force, cudaStream_t stream) {
  TrajTcArgs P;
  traj_tc_args(P, sig, n_sig, rirs, n_points, n_mics, L);
  P.out = out;
  P.part = partial;
  const int n_ctas = traj_tc_plan(P, num_sms, force);
  if (n_ctas <= 0) return cudaErrorInvalidValue;
  bool split = false;
  for (int t = 0; t < P.n_tiles && !split; t++) split = P.cta_first[t + 1] - P.cta_first[t] > 1;
  if (split && !partial) return cudaErrorInvalidValue;
  // TMA for the RIR windows when every 8-column group of a tile is 8 consecutive mics of one block
  static const bool no_tma = [] {
    const char* e = getenv("GPURIR_TRAJ_NO_TMA");  // A/B: register-fed B
    return e && e[0] == '1';
  }();
  const bool tma = !no_tma && (n_mics % 8) == 0 && tc_tensor_map_encoder() != nullptr;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof(tmap));
  if (tma) {
    const cuuint64_t dims[2] = {(cuuint64_t)L, (cuuint64_t)n_points * (cuuint64_t)n_mics};
    const cuuint64_t strides[1] = {(cuuint64_t)L * sizeof(float)};
    P.tma_rows = (n_mics % 32) == 0 ? 32 : 8;
    const cuuint32_t box[2] = {32, (cuuint32_t)P.tma_rows}, estr[2] = {1, 1};
    const CUresult r = tc_tensor_map_encoder()(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(rirs), dims,
                                               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  const size_t smem = (size_t)kTcSmemBytes;
  static unsigned long long attr_done = 0;  // bit per device: the dynamic shared-memory limits are set
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  if (dev >= 64 || !(__atomic_load_n(&attr_done, __ATOMIC_ACQUIRE) & (1ull << dev))) {
    e0 = cudaFuncSetAttribute(traj_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e0 == cudaSuccess)
      e0 = cudaFuncSetAttribute(traj_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e0 != cudaSuccess) return e0;
    if (dev < 64) __atomic_fetch_or(&attr_done, 1ull << dev, __ATOMIC_RELEASE);
  }
  if (tma)
    traj_tc_kernel<true><<<n_ctas, kTcThreads, smem, stream>>>(P, tmap);
  else
    traj_tc_kernel<false><<<n_ctas, kTcThreads, smem, stream>>>(P, tmap);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !split) return e;
  traj_reduce_kernel<<<dim3(kTcN * kTcM / 256, (unsigned)P.n_tiles), 256, 0, stream>>>(P);
  return cudaGetLastError();
}

}  // namespace gpurir

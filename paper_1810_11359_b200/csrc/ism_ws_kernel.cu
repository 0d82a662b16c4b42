// ism_ws_kernel.cu — persistent, warp-specialised ISM kernel for large batches
// (hot-path rows a1-a5 of SURVEY.md §8(a); same mathematics as ism_kernel.cu).
//
// One CTA per SM loops over (RIR, 512-sample tile) work items taken heaviest-first
// from a global counter.  Inside the CTA:
//   producer warps (16): enumerate the shell images of a tile column by column
//     (exact n_z ranges), compute each image's parameters in registers
//     (Eqs. 1-4; fp64 delay), append compact records to a
//     private window, stable-sort the window by delay bin and publish it into
//     one of two shared buffers;
//   consumer warps (16): wait for a published buffer, accumulate their four
//     8-sample sub-tiles from the contiguous record range of their bins
//     (Eqs. 5-6), release the buffer, and write the tile when its last window
//     has been consumed.
// Producer -> consumer hand-off uses named barriers (bar.arrive / bar.sync),
// so emission and sorting of window i+1 overlap the accumulation of window i
// and the consumer warps never wait on producer-internal phases.
#include <cuda_fp16.h>

#include "ism_common.cuh"

namespace gpurir {

#ifndef GPURIR_WS_CTAS_PER_SM
#define GPURIR_WS_CTAS_PER_SM 2
#endif
constexpr int kWsCtasPerSm = GPURIR_WS_CTAS_PER_SM;  // persistent CTAs per SM (1: 16P+16C, 2: 8P+8C each)
#ifndef GPURIR_WS_PW
#define GPURIR_WS_PW (16 / GPURIR_WS_CTAS_PER_SM)
#endif
constexpr int kPW = GPURIR_WS_PW;            // producer warps
constexpr int kCW = 32 / kWsCtasPerSm - kPW; // consumer warps
constexpr int kPT = kPW * 32;                // producer threads
constexpr int kWsThreads = (kPW + kCW) * 32; // 1024 / kWsCtasPerSm
constexpr int kWsSub = 4 * kWsCtasPerSm;     // 8-sample sub-tiles per consumer warp
constexpr int kWsTC = kCW * kWsSub * kS;     // 512 samples per tile
#ifndef GPURIR_WS_CAP
#define GPURIR_WS_CAP (4096 / GPURIR_WS_CTAS_PER_SM)
#endif
#ifndef GPURIR_WS_NBUF
#define GPURIR_WS_NBUF 3
#endif
// setmaxnreg split of the per-CTA register pool (kPW, kCW warps; 0 disables):
// kPW * PROD + kCW * CONS must equal (kPW + kCW) * 64.  Measured on cfg3: 80/48 -1.8 %, 88/40 -8.6 %
// (the consumer loop loses ILP), so it is off by default.
#ifndef GPURIR_WS_PROD_REGS
#define GPURIR_WS_PROD_REGS 0
#define GPURIR_WS_CONS_REGS 64
#endif
template <int MODE> struct WsCap { static constexpr int v = MODE == 1 ? GPURIR_WS_CAP / 2 : GPURIR_WS_CAP; };  // records per window
constexpr int kWsColBatch = kPT;             // columns per enumeration batch
constexpr int kBzMax = 1024;                 // z-factor table entries
static_assert(kWsTC == kTCPersistent, "tile size shared with the host planner");

constexpr int kNBuf = GPURIR_WS_NBUF;  // published window buffers (producers may run kNBuf - 1 windows ahead)
constexpr int kBarFull0 = 1;   // + buffer: producers arrive, consumers sync
constexpr int kBarEmpty0 = kBarFull0 + kNBuf;   // + buffer: consumers arrive, producers sync
constexpr int kBarProd = kBarEmpty0 + kNBuf;    // producer-internal

constexpr int kWinLast = 1, kWinTerminate = 2;

#ifdef GPURIR_WS_PROF  // profiling build only (tools/ws_prof.py): per-role cycle counters
__device__ unsigned long long g_ws_prof[64];
#define WS_T0(v) const long long v = clock64()
#define WS_ADD(i, v) prof[i] += (unsigned long long)(clock64() - (v))
#else
#define WS_T0(v)
#define WS_ADD(i, v)
#endif

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  unsigned a = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned a = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct WsStage {        // next work item's inputs, prefetched with cp.async by warp 0
  BatchJob job;          // batch call
  float pos[12];         // single-room call: src[3], rcv[3], orv[3], ors[3]
  long long wi;          // work index
  int2 jt;               // (job, tile) of a batch work item
};

// Work order: heaviest (latest) tiles first, which balances the tail of the persistent loop.  The
// alternative GPURIR_WS_DEALT deals heavy and light items alternately (measured 0.3 % slower on cfg3).
__device__ __forceinline__ long long ws_order(long long wi, long long n) {
#ifdef GPURIR_WS_DEALT
  return (wi & 1) ? n - 1 - (wi >> 1) : (wi >> 1);
#else
  (void)n;
  return wi;
#endif
}

// Single-room call: work position -> (RIR, tile).
#ifdef GPURIR_WS_RIR_MAJOR
// RIR-major: the tiles of one RIR are consecutive positions, latest (heaviest) first, so every CTA sees a
// mix of tile shapes (producer-heavy thin late shells, consumer-heavy middle tiles) at all times.
__device__ __forceinline__ int ws_tile(long long pos, const IsmArgs& A) { return A.nTiles - 1 - (int)(pos % A.nTiles); }
__device__ __forceinline__ int ws_rir(long long pos, const IsmArgs& A) { return (int)(pos / A.nTiles); }
#else
// tile-major: position 0..M-1 = the latest (heaviest) tile of every RIR, then the next tile, ...
__device__ __forceinline__ int ws_tile(long long pos, const IsmArgs& A) { return A.nTiles - 1 - (int)(pos / A.M); }
__device__ __forceinline__ int ws_rir(long long pos, const IsmArgs& A) { return (int)(pos % A.M); }
#endif

// Warp 0 of the producers: issue the asynchronous loads of work item wi's per-RIR inputs into stage.
__device__ __forceinline__ void ws_prefetch(const IsmArgs& A, long long wi, long long n_work, WsStage& st, int lane) {
  if (lane == 0) st.wi = wi;
  if (wi >= n_work) return;
  if (A.jobs) {
    int2 jt = A.tiles[ws_order(wi, n_work)];  // dependent: the job index selects the record to stage
    if (lane == 0) st.jt = jt;
    constexpr int n16 = (int)(sizeof(BatchJob) / 16);
    if (lane < n16) cp_async16(reinterpret_cast<char*>(&st.job) + 16 * lane, reinterpret_cast<const char*>(A.jobs + jt.x) + 16 * lane);
  } else {
    const int m = ws_rir(ws_order(wi, n_work), A);
    const int ms = m / A.M_rcv, mr = m % A.M_rcv;
    if (lane < 3) cp_async4(&st.pos[lane], A.pos_src + 3 * ms + lane);
    else if (lane < 6) cp_async4(&st.pos[lane], A.pos_rcv + 3 * mr + (lane - 3));
    else if (lane < 9 && A.orv) cp_async4(&st.pos[lane], A.orv + 3 * mr + (lane - 6));
    else if (lane < 9) st.pos[lane] = 0.f;
    else if (lane < 12 && A.ors) cp_async4(&st.pos[lane], A.ors + 3 * ms + (lane - 9));
    else if (lane < 12) st.pos[lane] = 0.f;
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

struct WsColRec {  // 32 B
  double rho2;     // (x_n - x_r)^2 + (y_n - y_r)^2
  float bxy;       // signed beta product of the x and y walls (C2)
  float cdot;      // (x_n - x_r) o_x + (y_n - y_r) o_y (polar pattern, C4)
  int r1lo, r2lo;  // n_z ranges [r1lo, r1lo + r1n), [r2lo, ...)
  int r1n;
  float sdot;      // column part of the source directivity (src_col_dot, f3)
};

struct WsTile {
  RirGeom g;
  double dlo2, dhi2, invLz, offE, offO;
  long long row;
  int m, t0, te, tc, nx0, ny0, NX, ncols, zl, zh;
  float xrel_max, invNX;
  int use_bz;
};

struct WinInfo {
  long long row;
  int t0, te, nbins, flags;
};


template <int MODE>
struct WsSmem {
  WsTile ti;
  WsStage stage;
  int next_work;
  WsColRec col[kWsColBatch];
  int colpre[kWsColBatch];
  float2 rec[WsCap<MODE>::v];
  float recA[MODE == 1 ? WsCap<MODE>::v : 1];
  uint8_t bin[WsCap<MODE>::v];
  uint16_t rank[WsCap<MODE>::v];  // rank of a record among its warp segment's records of the same bin
  int warpcnt[kPW][kMaxBins];
  int pbinstart[kMaxBins + 1];
  int scan_tmp[kPW];
  float bz[kBzMax];
  float4 sorted[kNBuf][MODE == 1 ? WsCap<MODE>::v + 8 : WsCap<MODE>::v / 2 + 8];
  int binstart[kNBuf][kMaxBins + 1];
  WinInfo win[kNBuf];
  float2 cacc[kCW][kWsSub][32];  // consumer accumulators (kept in smem so the tap loop can unroll 4 pairs)
};

// z-axis factor of beta_n (C2): signed beta_z0^|floor(n/2)| beta_z1^|ceil(n/2)|
__device__ __forceinline__ float z_factor(int nz, const RirGeom& g) {
  uint32_t sgn = 0;
  bool zero = false;
  float lz = axis_beta(nz, 2, g, sgn, zero);
  float v = zero ? 0.f : ex2_approx(lz);
  return sgn ? -v : v;
}

template <int MODE>
__global__ void __launch_bounds__(kWsThreads, kWsCtasPerSm) ism_ws_kernel(IsmArgs A, long long n_work, int* work_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WsSmem<MODE>& sm = *reinterpret_cast<WsSmem<MODE>*>(smem_raw);
  float2* lut = reinterpret_cast<float2*>(smem_raw + sizeof(WsSmem<MODE>));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float H = A.H;

  if (MODE == 1) {  // LUT table -> shared memory (once per persistent CTA)
    int n = A.lut_rows * A.lut_cols;
    for (int i = tid; i < n; i += kWsThreads) lut[i] = A.lut[i];
  }
  __syncthreads();

  if (warp < kPW) {
    // =========================== producers ===========================
#if GPURIR_WS_PROD_REGS > 0
    // rebalance the CTA's register pool: producers (fp64 image maths) up, consumers (FFMA2 loop) down
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(GPURIR_WS_PROD_REGS));
#endif
    const int ptid = tid;
    const unsigned lt = (1u << lane) - 1u;
    const double fs_over_c = A.fs_over_c;
    const double sc2 = fs_over_c * fs_over_c;
    const float fs_over_c_4pi = (float)fs_over_c * 0.0795774715459476679f;
    // per-mode record scale folded into each column's beta product: Eq. 4's fs/(4 pi c) and, for the fp32 /
    // fp16 records, the hoisted sinc factor -1/pi and the tap-argument scale
    const float rec_scale = MODE == 0   ? fs_over_c_4pi * -0.318309886183790672f * A.invHs
                            : MODE == 2 ? fs_over_c_4pi * -0.318309886183790672f * (0.5f * A.invHs) * 1024.f
                                        : fs_over_c_4pi;
    int win_i = 0, filled = 0;

    // stable counting sort of rec[0, filled) by bin, then publish to buffer win_i % kNBuf
#ifdef GPURIR_WS_PROF
    unsigned long long prof[16] = {0};
#endif
    auto publish = [&](int flags, int nbins) {
      WS_T0(tp0);
      for (int i = ptid; i < kPW * kMaxBins; i += kPT) (&sm.warpcnt[0][0])[i] = 0;
      bar_sync(kBarProd, kPT);
      const int per_warp = (filled + kPW - 1) / kPW;
      const int wbeg = warp * per_warp, wend = min(filled, wbeg + per_warp);
      for (int r0 = wbeg; r0 < wend; r0 += 32) {  // pass 1: per-warp bin counts and stable ranks
        int r = r0 + lane;
        int b = r < wend ? (int)sm.bin[r] : (int)kDiscard;
        unsigned peers = __match_any_sync(0xffffffffu, b);
        if (b != kDiscard) {
          const int before = sm.warpcnt[warp][b];
          sm.rank[r] = (uint16_t)(before + __popc(peers & lt));
        }
        __syncwarp();
        if (b != kDiscard && (peers & lt) == 0) sm.warpcnt[warp][b] += __popc(peers);
        __syncwarp();
      }
      bar_sync(kBarProd, kPT);
      if (ptid < nbins) {
        int s = 0;
        for (int w = 0; w < kPW; w++) { int c = sm.warpcnt[w][ptid]; sm.warpcnt[w][ptid] = s; s += c; }
        sm.pbinstart[ptid] = s;
      }
      bar_sync(kBarProd, kPT);
      if (warp == 0) {
        int carry = 0;
        for (int b0 = 0; b0 < nbins; b0 += 32) {
          int b = b0 + lane;
          int v = b < nbins ? sm.pbinstart[b] : 0;
          int x = warp_incl_scan(v, lane);
          if (b < nbins) sm.pbinstart[b] = carry + x - v;
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) sm.pbinstart[nbins] = carry;
      }
      const int buf = win_i % kNBuf;
      WS_T0(te0);
      if (win_i >= kNBuf) bar_sync(kBarEmpty0 + buf, kWsThreads);  // consumers released this buffer
      else bar_sync(kBarProd, kPT);
      WS_ADD(1, te0);
      float4* sorted = sm.sorted[buf];
      for (int r = wbeg + lane; r < wend; r += 32) {  // pass 2: scatter (no warp collectives)
        const int b = (int)sm.bin[r];
        if (b != kDiscard) {
          const int pos = sm.pbinstart[b] + sm.warpcnt[warp][b] + (int)sm.rank[r];
          const float2 rc = sm.rec[r];
          if (MODE == 1) {
            sorted[pos] = make_float4(rc.x, rc.y, sm.recA[r], 0.f);
          } else {  // pair layout: sorted[p>>1] = (nxv_even, nxv_odd, C_even, C_odd)
            float* pp = reinterpret_cast<float*>(&sorted[pos >> 1]);
            pp[pos & 1] = rc.x;
            pp[2 + (pos & 1)] = rc.y;
          }
        }
      }
      const int ntot = sm.pbinstart[nbins];
      if (ptid < 8) {  // dummy records after the last one (outside every window)
        int pos = ntot + ptid;
        if (MODE == 1) {
          sorted[pos] = make_float4(__int_as_float(0), 0.f, 0.f, 0.f);
        } else {
          float* pp = reinterpret_cast<float*>(&sorted[pos >> 1]);
          pp[pos & 1] = MODE == 3 ? -1.0e6f : -1.0e4f;  // outside every window / the texture
          pp[2 + (pos & 1)] = 0.f;
        }
      }
      for (int i = ptid; i <= nbins; i += kPT) sm.binstart[buf][i] = sm.pbinstart[i];
      if (ptid == 0) {
        WinInfo w;
        w.row = sm.ti.row; w.t0 = sm.ti.t0; w.te = sm.ti.te; w.nbins = nbins; w.flags = flags;
        sm.win[buf] = w;
      }
      bar_arrive(kBarFull0 + buf, kWsThreads);  // hand the buffer to the consumers
      bar_sync(kBarProd, kPT);                  // rec / warpcnt / pbinstart reusable
      win_i++;
      filled = 0;
      WS_ADD(0, tp0);
    };

    long long wi_pending = 0;  // warp 0, lane 0: the atomicAdd result for the item after the current one
    if (warp == 0) {
      long long wi0 = 0;
      if (lane == 0) wi0 = atomicAdd(work_counter, 1);
      wi0 = __shfl_sync(0xffffffffu, wi0, 0);
      ws_prefetch(A, wi0, n_work, sm.stage, lane);
    }
    for (;;) {
      WS_T0(ts0);
      if (warp == 0) {
        cp_async_wait_all();
        __syncwarp();
        if (lane == 0) {
          const long long wi = sm.stage.wi;
          sm.next_work = (int)min(wi, n_work);
          if (wi < n_work) {
            wi_pending = atomicAdd(work_counter, 1);  // consumed at the end of this tile (latency hidden)
            WsTile& T = sm.ti;
            int m, tile, nISM;
            long long row;
            const float zero3[3] = {0.f, 0.f, 0.f};
            if (A.jobs) {
              const BatchJob& J = sm.stage.job;
              m = sm.stage.jt.x; tile = sm.stage.jt.y;
              nISM = J.nISM;
              row = J.out_offset;
              geom_from(J.L, J.src, J.rcv, J.orv, J.nb, J.pattern, J.ors, J.spkr_pattern, J.lb, J.neg, J.zero, T.g,
                        A.status);
            } else {
              const long long pos = ws_order(wi, n_work);
              tile = ws_tile(pos, A);
              m = ws_rir(pos, A);
              nISM = A.nISM;
              row = (long long)m * A.row_stride;
              geom_from(A.L, sm.stage.pos, sm.stage.pos + 3, A.orv ? sm.stage.pos + 6 : zero3, A.nb, A.pattern,
                        A.ors ? sm.stage.pos + 9 : zero3, A.spkr_pattern, A.lb, A.neg, A.zero, T.g, A.status);
            }
            T.m = m; T.row = row;
            T.t0 = tile * kWsTC;
            T.te = min(T.t0 + kWsTC, nISM);
            T.tc = T.t0 + kWsTC / 2;
            T.invLz = 1.0 / T.g.L[2];
            T.offE = T.g.s[2] - T.g.r[2];
            T.offO = -T.g.s[2] - T.g.r[2];
            double xlo = (double)T.t0 - H, xhi = (double)(T.te - 1) + H;
            double dlo = xlo > 0.0 ? xlo * A.c_over_fs : 0.0;
            double dhi = xhi * A.c_over_fs;
            T.dlo2 = dlo * dlo;
            T.dhi2 = dhi * dhi;
            T.xrel_max = (float)(T.te - 1 - T.t0) + 2.f * H;
            int lo[2], hi[2];
            for (int ax = 0; ax < 2; ax++) {
              double L = T.g.L[ax], r = T.g.r[ax];
              int a = (int)floor((r - dhi) / L) - 1, b = (int)floor((r + dhi) / L) + 1;
              lo[ax] = max(a, T.g.nlo[ax]);
              hi[ax] = min(b, T.g.nhi[ax] - 1);
            }
            T.nx0 = lo[0]; T.ny0 = lo[1];
            T.NX = max(0, hi[0] - lo[0] + 1);
            T.ncols = T.NX * max(0, hi[1] - lo[1] + 1);
            T.invNX = T.NX > 0 ? 1.f / (float)T.NX : 0.f;
            T.zl = T.g.nlo[2];
            T.zh = T.g.nhi[2] - 1;
            T.use_bz = (T.zh - T.zl + 1) <= kBzMax;
          }
        }
      }
      bar_sync(kBarProd, kPT);
      if ((long long)sm.next_work >= n_work) break;
      bar_sync(kBarProd, kPT);
      WS_ADD(2, ts0);
      const WsTile& T = sm.ti;
      const RirGeom& g = T.g;
      const int nbins = (int)ceilf(((float)kWsTC + 2.f * H) / (float)kS) + 1;
      if (T.use_bz)
        for (int i = ptid; i <= T.zh - T.zl; i += kPT) sm.bz[i] = z_factor(T.zl + i, g);
      // (the first column batch below syncs before any bz read)

      for (int qb = 0; qb < T.ncols; qb += kWsColBatch) {
        WS_T0(tc0);
        int cnt = 0;
        {
          const int q = qb + ptid;
          WsColRec cr;
          cr.r1lo = 0; cr.r2lo = 0; cr.r1n = 0; cr.rho2 = 0.0; cr.bxy = 0.f; cr.cdot = 0.f; cr.sdot = 0.f;
          if (q < T.ncols) {
            const int qy = (int)(((float)q + 0.5f) * T.invNX);  // q / NX, exact for q < 2^20
            const int nx = T.nx0 + (q - qy * T.NX), ny = T.ny0 + qy;
            const double dx = image_coord(nx, g.L[0], g.s[0]) - g.r[0];
            const double dy = image_coord(ny, g.L[1], g.s[1]) - g.r[1];
            const double rho2 = dx * dx + dy * dy;
            cr.rho2 = rho2;
            cr.cdot = (float)dx * g.o[0] + (float)dy * g.o[1];
            cr.sdot = src_col_dot(nx, ny, (float)dx, (float)dy, g);
            uint32_t sgn = 0; bool zero = false;
            float lxy = axis_beta(nx, 0, g, sgn, zero) + axis_beta(ny, 1, g, sgn, zero);
            float bxy = zero ? 0.f : ex2_approx(lxy);
            cr.bxy = (sgn ? -bxy : bxy) * rec_scale;
            if (rho2 < T.dhi2) {
              // shell bounds along z: fp32 square roots suffice (an image misplaced by their rounding sits on the
              // shell edge, where its window weight is ~0); the ranges below are exact for these bounds
              const double zhi = (double)sqrtf((float)(T.dhi2 - rho2));
              const double zlo = T.dlo2 > rho2 ? (double)sqrtf((float)(T.dlo2 - rho2)) : 0.0;
              int pa, pb, na, nbz;
              z_range(g, T.invLz, zlo, zhi, pa, pb);
              z_range(g, T.invLz, -zhi, -zlo, na, nbz);
              if (nbz >= pa - 1) { pa = min(pa, na); na = 1; nbz = 0; }
              pa = max(pa, T.zl); pb = min(pb, T.zh);
              na = max(na, T.zl); nbz = min(nbz, T.zh);
              int n1 = max(0, pb - pa + 1), n2 = max(0, nbz - na + 1);
              cr.r1lo = pa; cr.r1n = n1; cr.r2lo = na;
              cnt = n1 + n2;
            }
          }
          sm.col[ptid] = cr;
        }
        // block scan over the producer threads
        int x = warp_incl_scan(cnt, lane);
        if (lane == 31) sm.scan_tmp[warp] = x;
        bar_sync(kBarProd, kPT);
        int add = 0;
        for (int w = 0; w < warp; w++) add += sm.scan_tmp[w];
        sm.colpre[ptid] = x + add;
        bar_sync(kBarProd, kPT);
        const int total = sm.colpre[kWsColBatch - 1];
        WS_ADD(3, tc0);
        WS_T0(ti0);

        for (int base = 0; base < total;) {
          const int take = min(WsCap<MODE>::v - filled, total - base);
          const int R = (take + kPT - 1) / kPT;
          const int g0 = base + ptid * R, g1 = min(g0 + R, base + take);
          if (g0 < g1) {
            int lo = 0, hi = kWsColBatch - 1;  // first column with colpre > g0
            while (lo < hi) {
              int mid = (lo + hi) >> 1;
              if (sm.colpre[mid] > g0) hi = mid; else lo = mid + 1;
            }
            int j = lo;
            int before = j > 0 ? sm.colpre[j - 1] : 0;
            int boundary = sm.colpre[j];
            // tile constants in registers (shared-memory reads would be re-issued per image)
            const double Lz = g.L[2], offE = T.offE, offO = T.offO;
            const float Lzf = (float)Lz, offEf = (float)offE, offOf = (float)offO;
            const int tc = T.tc, zl = T.zl;
            const bool use_bz = T.use_bz;
            const float xmax = T.xrel_max, oz = g.o[2], ga = g.a, fsc = (float)fs_over_c;
            const bool dir_src = g.as != 1.f;  // directional source (f3): tile-uniform branch
            // Two images per iteration: all shared loads first, then both images' arithmetic (independent,
            // so the scheduler interleaves the two dependency chains), then the stores.
            for (int gi = g0; gi < g1; gi += 2) {
              while (gi >= boundary) { before = boundary; j++; boundary = sm.colpre[j]; }
              const int jA = j, lA = gi - before;
              const bool hasB = gi + 1 < g1;
              if (hasB) { while (gi + 1 >= boundary) { before = boundary; j++; boundary = sm.colpre[j]; } }
              const int jB = j, lB = gi + 1 - before;
              const WsColRec crA = sm.col[jA], crB = sm.col[jB];
              int nz[2], odd[2];
              nz[0] = lA < crA.r1n ? crA.r1lo + lA : crA.r2lo + (lA - crA.r1n);
              nz[1] = lB < crB.r1n ? crB.r1lo + lB : crB.r2lo + (lB - crB.r1n);
              float bz[2];
#pragma unroll
              for (int e = 0; e < 2; e++) {
                odd[e] = nz[e] & 1;
                bz[e] = use_bz ? sm.bz[min(max(nz[e] - zl, 0), kBzMax - 1)] : z_factor(nz[e], g);
              }
              float2 rec[2];
              float recA[2];
              uint8_t bb[2];
#pragma unroll
              for (int e = 0; e < 2; e++) {
                const WsColRec& cr = e ? crB : crA;
                // Eq. 1 along z: even nz -> nz L + s, odd nz -> (nz + 1) L - s; Delta_z = z_n - z_r
                const int nzo = nz[e] + odd[e];
                const double dz = fma(int_to_double(nzo), Lz, odd[e] ? offO : offE);
                const double x2 = fma(dz, dz, cr.rho2) * sc2;  // (d fs / c)^2
                if (x2 == 0.0 && (e == 0 || hasB)) atomicOr(A.status, kStatusDegenerate);
                // branch-free from here: culled records are computed and flagged with kDiscard
                float x0f, rx;                              // rx = rsqrt(x^2) = 1/x, so 1/d = fs rx / c
                float xr = delay_rel(x2, tc, x0f, rx);
                const float xrel = xr + (float)(kWsTC / 2) + H;  // x - (t0 - H)
                const bool keep = (x2 != 0.0) && (xrel > 0.f) && (xrel < xmax);
                bb[e] = keep ? (uint8_t)floor_div8(xrel) : kDiscard;
                const float dzf = fmaf((float)nzo, Lzf, odd[e] ? offOf : offEf);  // fp32 Delta_z (directivity)
                const float cth = fmaf(dzf, oz, cr.cdot) * (fsc * rx);
                float gain = ga + (1.f - ga) * cth;
                if (dir_src) gain *= src_gain(cr.sdot, odd[e], dzf, fsc * rx, g);
                const float amp = cr.bxy * bz[e] * gain * rx;  // Eq. 4 (times rec_scale)
                recA[e] = 0.f;
                if (MODE == 1) {
                  float xq = xr * (float)A.lutQ;
                  float fiq = floorf(xq);
                  float phi = xq - fiq;
                  int iq1 = (int)fiq + 1;
                  int php = iq1 & (A.lutQ - 1);
                  int aa = (iq1 - php) / A.lutQ;
                  int ph = (A.lutQ - php) & (A.lutQ - 1);
                  int jsh = aa + (php > 0 ? 1 : 0);
                  rec[e] = make_float2(__int_as_float(ph * A.lut_cols + A.lut_joff - jsh), phi);
                  recA[e] = amp;
                } else if (MODE == 3) {
                  rec[e] = make_float2(fmaf(-xr, A.texQ, A.tex_off), amp);  // coordinate offset, amplitude
                } else {
                  int jodd;
                  const float fj = floor_parity(xr, jodd);
                  // exact integer delay (reading R3): move up by >= 1 ulp (floor unchanged; select, no branch)
                  xr = (xr == fj) ? xr + fmaxf(fabsf(xr) * 1.1920929e-7f, 9.5367432e-7f) : xr;
                  const float f = xr - fj;
                  float cc = amp * sinpi01(f);  // C' = -A sin(pi f) / pi (scaled), rec_scale
                  if (jodd) cc = -cc;
                  rec[e] = make_float2(-xr * (MODE == 0 ? A.invHs : 0.5f * A.invHs), cc);
                }
              }
              const int dst = filled + (gi - base);
              sm.rec[dst] = rec[0];
              if (MODE == 1) sm.recA[dst] = recA[0];
              sm.bin[dst] = bb[0];
              if (hasB) {
                sm.rec[dst + 1] = rec[1];
                if (MODE == 1) sm.recA[dst + 1] = recA[1];
                sm.bin[dst + 1] = bb[1];
              }
            }
          }
          filled += take;
          base += take;
          if (filled == WsCap<MODE>::v) {
            bar_sync(kBarProd, kPT);
            publish(0, nbins);
          }
        }
        bar_sync(kBarProd, kPT);  // column records are replaced by the next batch
        WS_ADD(4, ti0);  // includes the publishes of full windows (also counted in [0])
      }
      if (warp == 0) {  // stage the next work item while the last window is sorted and published
        const long long wn = __shfl_sync(0xffffffffu, wi_pending, 0);
        ws_prefetch(A, wn, n_work, sm.stage, lane);
      }
      bar_sync(kBarProd, kPT);
      publish(kWinLast, nbins);  // the tile's last window (possibly empty)
    }
    publish(kWinTerminate, 1);
    // match the consumers' releases of the last kNBuf buffers
    for (int w = max(0, win_i - kNBuf); w < win_i; w++) bar_sync(kBarEmpty0 + (w % kNBuf), kWsThreads);
#ifdef GPURIR_WS_PROF
    if (lane == 0)
      for (int i = 0; i < 8; i++) atomicAdd(&g_ws_prof[i], prof[i]);
#endif
  } else {
    // =========================== consumers ===========================
#if GPURIR_WS_PROD_REGS > 0
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(GPURIR_WS_CONS_REGS));
#endif
    const int cw = warp - kPW;
    const int grp = lane >> 3, li = lane & 7;
    float2 (*acc)[32] = sm.cacc[cw];
#pragma unroll
    for (int s = 0; s < kWsSub; s++) acc[s][lane] = make_float2(0.f, 0.f);
    int win_i = 0;
#ifdef GPURIR_WS_PROF
    unsigned long long prof[32] = {0};
#endif
    for (;;) {
      const int buf = win_i % kNBuf;
      WS_T0(tf0);
      bar_sync(kBarFull0 + buf, kWsThreads);
      const WinInfo w = sm.win[buf];
#ifdef GPURIR_WS_PROF
      const int tb = min(w.t0 / kWsTC, 7);
      prof[tb] += (unsigned long long)(clock64() - tf0);
      prof[24 + tb] += 1;
#endif
      WS_T0(tw0);
      if (w.flags & kWinTerminate) {
        bar_arrive(kBarEmpty0 + buf, kWsThreads);
        break;
      }
      const float4* sorted = sm.sorted[buf];
#pragma unroll 1
      for (int s = 0; s < kWsSub; s++) {
        const int sub = s * kCW + cw;  // interleaved: every warp gets early and late sub-tiles of the tile
        if (sub * kS >= w.te - w.t0) break;  // past the end of a partial (last) tile
        const int kf = sub * kS + li - kWsTC / 2;  // sample relative to the tile centre
        const int ra = sm.binstart[buf][sub], rb = sm.binstart[buf][min(sub + A.nbw, w.nbins)];
        if (MODE == 0) {
          const TapConst K = make_tap_const(A, (float)kf * A.invHs);
          const float4* pp = sorted + ((ra & ~1) >> 1) + grp;  // record pairs, group grp, stride kG
          const float4* pend = sorted + ((rb + 1) >> 1);
          acc[s][lane] = tap_loop(pp, pend, K, acc[s][lane]);
        } else if (MODE == 2) {
          TapConstH K;
          const float kx = (float)kf * (0.5f * A.invHs);
          K.kx2 = make_float2(kx, kx);
          K.c6 = __float2half2_rn(A.hc[2]); K.c4 = __float2half2_rn(A.hc[1]);
          K.c2 = __float2half2_rn(A.hc[0]); K.c0 = __float2half2_rn(1.f);
          K.xcl = __float2half2_rn(A.x2clamp);
          const float4* pp = sorted + ((ra & ~1) >> 1) + grp;
          const float4* pend = sorted + ((rb + 1) >> 1);
          acc[s][lane] = tap_loop_h(pp, pend, K, acc[s][lane]);
        } else if (MODE == 3) {
          const float4* pp = sorted + ((ra & ~1) >> 1) + grp;
          const float4* pend = sorted + ((rb + 1) >> 1);
          acc[s][lane] = tap_loop_tex(pp, pend, (cudaTextureObject_t)A.tex, (float)kf * A.texQ, acc[s][lane]);
        } else {
          float a = acc[s][lane].x;
          for (int j = ra + grp; j < rb; j += kG) {
            float4 rc = sorted[j];
            int idx = __float_as_int(rc.x) + kf;
            float2 d = lut[idx];
            a = fmaf(rc.z, fmaf(rc.y, d.y, d.x), a);
          }
          acc[s][lane].x = a;
        }
      }
      bar_arrive(kBarEmpty0 + buf, kWsThreads);  // buffer consumed
      if (w.flags & kWinLast) {
#pragma unroll
        for (int s = 0; s < kWsSub; s++) {
          const float2 as = acc[s][lane];
          float a = as.x + as.y;
          a += __shfl_xor_sync(0xffffffffu, a, 8);
          a += __shfl_xor_sync(0xffffffffu, a, 16);
          const int kf = (s * kCW + cw) * kS + li - kWsTC / 2;
          if (MODE == 0) { if (kf & 1) a = -a; }
          else if (MODE == 2) { a *= (1.f / 1024.f); if (kf & 1) a = -a; }
          const int k = w.t0 + (s * kCW + cw) * kS + li;
          if (grp == 0 && k < w.te) A.out[w.row + k] = a;
          acc[s][lane] = make_float2(0.f, 0.f);
        }
      }
#ifdef GPURIR_WS_PROF
      prof[8 + tb] += (unsigned long long)(clock64() - tw0);
#endif
      win_i++;
    }
#ifdef GPURIR_WS_PROF
    if (lane == 0)
      for (int i = 0; i < 32; i++) if (prof[i]) atomicAdd(&g_ws_prof[16 + i], prof[i]);
#endif
  }
}

#ifdef GPURIR_WS_PROF
extern "C" int gpurir_debug_ws_prof(unsigned long long* out64, int reset) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out64, g_ws_prof, sizeof(g_ws_prof)) != cudaSuccess) return 5;
  if (reset) {
    unsigned long long z[64] = {0};
    cudaMemcpyToSymbol(g_ws_prof, z, sizeof(z));
  }
  return 0;
}
#endif

size_t ism_ws_smem_bytes(int mode, int lut_rows, int lut_cols) {
  switch (mode) {
    case 0: return sizeof(WsSmem<0>);
    case 1: return sizeof(WsSmem<1>) + (size_t)lut_rows * lut_cols * sizeof(float2);
    case 3: return sizeof(WsSmem<3>);
    default: return sizeof(WsSmem<2>);
  }
}

template <int MODE>
static cudaError_t launch_ws_mode(const IsmArgs& A, long long n_work, int* counter, int grid, size_t smem,
                                  cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(ism_ws_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ism_ws_kernel<MODE><<<grid, kWsThreads, smem, stream>>>(A, n_work, counter);
  return cudaGetLastError();
}

cudaError_t launch_ism_ws(const IsmArgs& A, int mode, long long n_work, int* counter, int num_sms,
                          cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int), stream);
  if (e != cudaSuccess) return e;
  const long long slots = (long long)num_sms * kWsCtasPerSm;
  int grid = (int)(n_work < slots ? n_work : slots);
  size_t smem = ism_ws_smem_bytes(mode, A.lut_rows, A.lut_cols);
  switch (mode) {
    case 0: return launch_ws_mode<0>(A, n_work, counter, grid, smem, stream);
    case 1: return launch_ws_mode<1>(A, n_work, counter, grid, smem, stream);
    case 3: return launch_ws_mode<3>(A, n_work, counter, grid, smem, stream);
    default: return launch_ws_mode<2>(A, n_work, counter, grid, smem, stream);
  }
}

}  // namespace gpurir

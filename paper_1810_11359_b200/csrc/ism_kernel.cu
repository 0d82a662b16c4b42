// ism_kernel.cu — fused image-parameter + delay-binning + RIR-accumulation kernel
// (hot-path rows a1, a2, a3, a4, a5 of SURVEY.md §8(a)) for sm_100a.
//
// What it computes (§2.1-2.2, Eqs. 1-6):
//   h[m][k] = sum_n A_n * delta'(k/fs - tau_n),   0 <= k < nISM,
//   A_n = beta_n g_n / (4 pi d_n), tau_n = d_n / c, delta' = Hann-windowed sinc of length T_w.
// How: one CTA owns a tile of kTC output samples of one RIR.
//  1. It enumerates only the lattice images whose window can touch the tile (a
//     spherical shell around the receiver), column by column (n_x, n_y), with the
//     n_z range of each column solved exactly (Delta_z is monotone in n_z).
//  2. Image parameters are computed in registers (fp64 delay, C1/C2/C4) and
//     written as compact records into a shared-memory window of kCap records;
//     windows are filled across column batches.
//  3. A stable counting sort bins the window's records by delay (deterministic).
//  4. Every warp accumulates its two 8-sample sub-tiles from the contiguous
//     record range of their bins: 4 lane groups x 2 packed (f32x2) records per
//     step, accumulators in registers, shuffle reduction at the end.
// Thread-block clusters split the columns of one tile across `split` CTAs
// whose partial tiles are summed through distributed shared memory (fixed order).
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include "ism_common.cuh"

namespace cg = cooperative_groups;

namespace gpurir {

constexpr int kSubPerWarp = kTC / (kWarps * kS);  // 8-sample sub-tiles per warp
static_assert(kSubPerWarp * kWarps * kS == kTC, "tile geometry");

// ----------------------------------------------------------------------------
// shared-memory layout
// ----------------------------------------------------------------------------
struct ColRec {         // one lattice column (n_x, n_y) of the current batch (32 B)
  double rho2;          // (x_n - x_r)^2 + (y_n - y_r)^2
  float cdot, sdot;     // column parts of the receiver / source directivity (C4; f3)
  float lxy;            // log2 |beta product| of the x and y walls
  int r1lo, r2lo;       // n_z ranges [r1lo, r1lo + r1n) then [r2lo, ...)
  uint32_t r1n_flags;   // r1n | sign << 30 | zero << 31
};

struct TileInfo {
  RirGeom g;
  double dlo2, dhi2;    // shell in distance^2
  double invLz;         // 1 / L_z
  int m, tile, t0, te, tc;
  int nx0, ny0, NX, ncols_mine;
  long long row;        // element offset of the RIR row
  float xrel_max;       // records with xrel in (0, xrel_max) are kept
  int nbins;
};

struct Smem {
  TileInfo ti;
  int colpre[kColBatch];          // inclusive prefix of candidate counts
  ColRec col[kColBatch];
  float2 rec[kCap];               // unsorted records: fp32/fp16 (-x/Hs, C'), LUT (rowbase, phi)
  float recA[kCap];               // LUT amplitude
  uint8_t bin[kCap];
  float4 sorted[kCap + 8];        // sorted records; fp32/fp16 modes pack pairs
  int warpcnt[kWarps][kMaxBins];  // per-warp bin counts -> offsets
  int binstart[kMaxBins + 1];
  int scan_tmp[kWarps];
  float outtile[kTC];
};

// Block-wide inclusive scan (kThreads values); returns the inclusive prefix for this thread.
__device__ __forceinline__ int block_incl_scan(int v, int* tmp) {
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = warp_incl_scan(v, lane);
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < kWarps ? tmp[lane] : 0;
    t = warp_incl_scan(t, lane);
    if (lane < kWarps) tmp[lane] = t;
  }
  __syncthreads();
  int r = x + (w > 0 ? tmp[w - 1] : 0);
  return r;
}

// ----------------------------------------------------------------------------
// The kernel
// ----------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) ism_kernel(IsmArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  float2* lut = reinterpret_cast<float2*>(smem_raw + sizeof(Smem));

  cg::cluster_group cluster = cg::this_cluster();
  const int P = (int)cluster.num_blocks();
  const int prank = (int)cluster.block_rank();
  const int cid = blockIdx.x / P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float H = A.H;

  // ---- tile setup (thread 0) ------------------------------------------------
  if (tid == 0) {
    TileInfo& T = sm.ti;
    int m, tile, nISM;
    long long row;
    if (A.jobs) {
      int2 jt = A.tiles[cid];
      m = jt.x; tile = jt.y;
      nISM = A.jobs[m].nISM;
      row = A.jobs[m].out_offset;
    } else {
      tile = A.nTiles - 1 - cid / A.M;  // heaviest (latest) tiles first
      m = cid % A.M;
      nISM = A.nISM;
      row = (long long)m * A.row_stride;
    }
    load_geom(A, m, T.g, A.status);
    T.m = m; T.tile = tile; T.row = row;
    T.t0 = tile * kTC;
    T.te = min(T.t0 + kTC, nISM);
    T.tc = T.t0 + kTC / 2;
    T.invLz = 1.0 / T.g.L[2];
    // shell: images with x in (t0 - H, te - 1 + H) can touch samples [t0, te)
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
    int NY = max(0, hi[1] - lo[1] + 1);
    long long ncols = (long long)T.NX * NY;
    T.ncols_mine = (int)((ncols - prank + P - 1) / P);
    if (T.ncols_mine < 0) T.ncols_mine = 0;
    T.nbins = (int)ceilf(((float)kTC + 2.f * H) / (float)kS) + 1;
  }
  if (MODE == 1) {  // LUT table -> shared memory
    int n = A.lut_rows * A.lut_cols;
    for (int i = tid; i < n; i += kThreads) lut[i] = A.lut[i];
  }
  __syncthreads();
  const TileInfo& T = sm.ti;
  const RirGeom& g = T.g;
  const int nbins = T.nbins;

  // ---- per-lane accumulation constants (two 8-sample sub-tiles per warp) ------
  const int grp = lane >> 3, li = lane & 7;
  int kfs[kSubPerWarp];
  float2 acc[kSubPerWarp];
#pragma unroll
  for (int s = 0; s < kSubPerWarp; s++) {
    kfs[s] = T.t0 + (s * kWarps + warp) * kS + li - T.tc;  // sample relative to tc
    acc[s] = make_float2(0.f, 0.f);
  }

  const double fs_over_c = A.fs_over_c;
  const double sc2 = fs_over_c * fs_over_c;
  const float fs_over_c_4pi = (float)fs_over_c * 0.0795774715459476679f;

  // ---- window processing: stable bin sort + accumulation -----------------------
  auto process_window = [&](int nw) {
    for (int i = tid; i < kWarps * kMaxBins; i += kThreads) (&sm.warpcnt[0][0])[i] = 0;
    __syncthreads();
    const int per_warp = (nw + kWarps - 1) / kWarps;
    const int wbeg = warp * per_warp, wend = min(nw, wbeg + per_warp);
    const unsigned lt = (1u << lane) - 1u;
    for (int r0 = wbeg; r0 < wend; r0 += 32) {
      int r = r0 + lane;
      int b = r < wend ? (int)sm.bin[r] : (int)kDiscard;
      unsigned peers = __match_any_sync(0xffffffffu, b);
      if (b != kDiscard && (peers & lt) == 0) sm.warpcnt[warp][b] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    if (tid < nbins) {  // per bin: prefix over warps
      int s = 0;
      for (int w = 0; w < kWarps; w++) { int c = sm.warpcnt[w][tid]; sm.warpcnt[w][tid] = s; s += c; }
      sm.binstart[tid] = s;  // bin total for now
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of bin totals (nbins <= 128)
      int carry = 0;
      for (int b0 = 0; b0 < nbins; b0 += 32) {
        int b = b0 + lane;
        int v = b < nbins ? sm.binstart[b] : 0;
        int x = warp_incl_scan(v, lane);
        if (b < nbins) sm.binstart[b] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) sm.binstart[nbins] = carry;
    }
    __syncthreads();
    for (int r0 = wbeg; r0 < wend; r0 += 32) {
      int r = r0 + lane;
      int b = r < wend ? (int)sm.bin[r] : (int)kDiscard;
      unsigned peers = __match_any_sync(0xffffffffu, b);
      if (b != kDiscard) {
        int pos = sm.binstart[b] + sm.warpcnt[warp][b] + __popc(peers & lt);
        float2 rc = sm.rec[r];
        if (MODE == 1) {
          sm.sorted[pos] = make_float4(rc.x, rc.y, sm.recA[r], 0.f);
        } else {  // pair layout: sorted[p>>1] = (nxv_even, nxv_odd, C_even, C_odd)
          float* pp = reinterpret_cast<float*>(&sm.sorted[pos >> 1]);
          pp[pos & 1] = rc.x;
          pp[2 + (pos & 1)] = rc.y;
        }
      }
      __syncwarp();
      if (b != kDiscard && (peers & lt) == 0) sm.warpcnt[warp][b] += __popc(peers);
      __syncwarp();
    }
    if (tid < 8) {  // dummy records after the last one (outside every window: v = kv - 1e4)
      int pos = sm.binstart[nbins] + tid;
      if (MODE == 1) {
        sm.sorted[pos] = make_float4(__int_as_float(0), 0.f, 0.f, 0.f);
      } else {
        float* pp = reinterpret_cast<float*>(&sm.sorted[pos >> 1]);
        pp[pos & 1] = MODE == 3 ? -1.0e6f : -1.0e4f;
        pp[2 + (pos & 1)] = 0.f;
      }
    }
    __syncthreads();

#pragma unroll
    for (int s = 0; s < kSubPerWarp; s++) {
      const int sub = s * kWarps + warp;  // interleaved sub-tiles (balances the t^2 image density)
      const int ra = sm.binstart[sub], rb = sm.binstart[min(sub + A.nbw, nbins)];
      if (MODE == 0) {
        // Eq. 5-6: acc += C' w(u) / v, v = (k - x)/Hs, w = Hann window (R5), C' = -A sin(pi f)/(pi Hs)
        const TapConst K = make_tap_const(A, (float)kfs[s] * A.invHs);
        const float4* pp = sm.sorted + ((ra & ~1) >> 1) + grp;  // record pairs, group grp, stride kG
        const float4* pend = sm.sorted + ((rb + 1) >> 1);
        acc[s] = tap_loop(pp, pend, K, acc[s]);
      } else if (MODE == 2) {
        // fp16 / half2: t - tau in fp32, window by the Eq. 11 polynomial
        // cos(pi x) at x = u / (2H) (reading C12), half2 Horner (Eq. 12), fp32 accumulation (C13).
        const float kx = (float)kfs[s] * (0.5f * A.invHs);
        const float2 kx2 = make_float2(kx, kx);
        const __half2 c6 = __float2half2_rn(A.hc[2]), c4 = __float2half2_rn(A.hc[1]);
        const __half2 c2 = __float2half2_rn(A.hc[0]), c0 = __float2half2_rn(1.f);
        const __half2 xcl = __float2half2_rn(A.x2clamp);
        __half2 acch = __float2half2_rn(0.f);
        float2 a2 = acc[s];
        int steps = 0;
        for (int j = (ra & ~1) + 2 * grp; j < rb; j += 2 * kG) {
          float4 pr = sm.sorted[j >> 1];
          float2 x = __fadd2_rn(kx2, make_float2(pr.x, pr.y));      // x' = (k - tau fs) / (2 Hs), fp32
          __half2 hx = __float22half2_rn(x);
          __half2 x2 = __hmin2(__hmul2(hx, hx), xcl);                // clamp: |u/(2H)| <= 1/2 (window edge)
          __half2 p = __hfma2(c6, x2, c4);
          p = __hfma2(p, x2, c2);
          p = __hfma2(p, x2, c0);                                    // cos(pi x), Eq. 11
          __half2 w = __hmul2(p, p);                                 // Hann window
          float2 r = make_float2(rcp_approx(x.x), rcp_approx(x.y));
          float2 q = __fmul2_rn(make_float2(pr.z, pr.w), r);         // bounded by ~A (scaled 2^10)
          acch = __hfma2(w, __float22half2_rn(q), acch);
          if (++steps == 8) {
            float2 f = __half22float2(acch);
            a2.x += f.x; a2.y += f.y;
            acch = __float2half2_rn(0.f);
            steps = 0;
          }
        }
        float2 f = __half22float2(acch);
        a2.x += f.x; a2.y += f.y;
        acc[s] = a2;
      } else if (MODE == 3) {
        // texture LUT (f2): hardware linear interpolation of the Eq. 9 table
        const float4* pp = sm.sorted + ((ra & ~1) >> 1) + grp;
        const float4* pend = sm.sorted + ((rb + 1) >> 1);
        acc[s] = tap_loop_tex(pp, pend, (cudaTextureObject_t)A.tex, (float)kfs[s] * A.texQ, acc[s]);
      } else {
        // LUT (Eq. 9): one table pair per tap, phase-major rows, linear interpolation
        float a = acc[s].x;
        for (int j = ra + grp; j < rb; j += kG) {
          float4 rc = sm.sorted[j];
          int idx = __float_as_int(rc.x) + kfs[s];
          float2 d = lut[idx];
          a = fmaf(rc.z, fmaf(rc.y, d.y, d.x), a);
        }
        acc[s].x = a;
      }
    }
    __syncthreads();  // records of this window are consumed
  };

  // ---- enumeration: column batches, candidate stream, windows of kCap records ----
  int filled = 0;
  for (int qb = 0; qb < T.ncols_mine; qb += kColBatch) {
    int cnt = 0;
    {
      int q = qb + tid;
      ColRec cr;
      cr.r1lo = 0; cr.r2lo = 0;
      int r1n = 0;
      uint32_t fl = 0;
      if (q < T.ncols_mine) {
        int ci = prank + P * q;
        int nx = T.nx0 + ci % T.NX, ny = T.ny0 + ci / T.NX;
        double dx = image_coord(nx, g.L[0], g.s[0]) - g.r[0];
        double dy = image_coord(ny, g.L[1], g.s[1]) - g.r[1];
        double rho2 = dx * dx + dy * dy;
        cr.rho2 = rho2;
        cr.cdot = (float)dx * g.o[0] + (float)dy * g.o[1];
        cr.sdot = src_col_dot(nx, ny, (float)dx, (float)dy, g);
        uint32_t sgn = 0; bool zero = false;
        cr.lxy = axis_beta(nx, 0, g, sgn, zero) + axis_beta(ny, 1, g, sgn, zero);
        fl = (sgn << 30) | (zero ? (1u << 31) : 0u);
        if (rho2 < T.dhi2) {
          double zhi = sqrt(T.dhi2 - rho2);
          double zlo = T.dlo2 > rho2 ? sqrt(T.dlo2 - rho2) : 0.0;
          int pa, pb, na, nbz;
          z_range(g, T.invLz, zlo, zhi, pa, pb);     // Delta_z in [zlo, zhi]
          z_range(g, T.invLz, -zhi, -zlo, na, nbz);  // Delta_z in [-zhi, -zlo]
          if (nbz >= pa - 1) { pa = min(pa, na); na = 1; nbz = 0; }  // sides touch (zlo ~ 0): merge
          const int zl = g.nlo[2], zh = g.nhi[2] - 1;
          pa = max(pa, zl); pb = min(pb, zh);
          na = max(na, zl); nbz = min(nbz, zh);
          int n1 = max(0, pb - pa + 1), n2 = max(0, nbz - na + 1);
          cr.r1lo = pa; r1n = n1; cr.r2lo = na;
          cnt = n1 + n2;
        }
      }
      cr.r1n_flags = (uint32_t)r1n | fl;
      sm.col[tid] = cr;
    }
    int incl = block_incl_scan(cnt, sm.scan_tmp);
    sm.colpre[tid] = incl;
    __syncthreads();
    const int total = sm.colpre[kColBatch - 1];

    for (int base = 0; base < total;) {
      const int take = min(kCap - filled, total - base);
      // ---- emission: contiguous candidate runs per thread, one binary search each ----
      const int R = (take + kThreads - 1) / kThreads;
      const int g0 = base + tid * R, g1 = min(g0 + R, base + take);
      if (g0 < g1) {
        int lo = 0, hi = kColBatch - 1;  // first column with colpre > g0
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (sm.colpre[mid] > g0) hi = mid; else lo = mid + 1;
        }
        int j = lo;
        int before = j > 0 ? sm.colpre[j - 1] : 0;
        for (int gi = g0; gi < g1; gi++) {
          while (sm.colpre[j] <= gi) { before = sm.colpre[j]; j++; }
          const ColRec& cr = sm.col[j];
          const int l = gi - before;
          const int r1n = (int)(cr.r1n_flags & 0x3FFFFFFFu);
          const int nz = l < r1n ? cr.r1lo + l : cr.r2lo + (l - r1n);
          const double dz = image_coord(nz, g.L[2], g.s[2]) - g.r[2];
          const double x2 = fma(dz, dz, cr.rho2) * sc2;  // (d fs / c)^2
          uint8_t b = kDiscard;
          float2 rec = make_float2(0.f, 0.f);
          float recA = 0.f;
          if (x2 == 0.0) {
            atomicOr(A.status, kStatusDegenerate);
          } else {
            float x0f;
            float xr = delay_rel(x2, T.tc, x0f);
            float xrel = xr + (float)(kTC / 2) + H;  // x - (t0 - H)
            if (xrel > 0.f && xrel < T.xrel_max) {
              b = (uint8_t)(int)(xrel * (1.f / (float)kS));
              // amplitude A = beta_n g / (4 pi d), 1/d = fs / (c x)     (Eq. 4, A16)
              const float rx = rcp_approx(x0f);
              uint32_t sgn = (cr.r1n_flags >> 30) & 1u;
              bool zero = (cr.r1n_flags >> 31) != 0;
              const float lz = axis_beta(nz, 2, g, sgn, zero);
              float bn = zero ? 0.f : ex2_approx(cr.lxy + lz);
              if (sgn) bn = -bn;
              const float cth = fmaf((float)dz, g.o[2], cr.cdot) * ((float)fs_over_c * rx);
              const float gain = (g.a + (1.f - g.a) * cth) * src_gain(cr.sdot, nz & 1, (float)dz, (float)fs_over_c * rx, g);
              const float amp = bn * gain * rx * fs_over_c_4pi;
              if (MODE == 1) {
                // Eq. 9 LUT: position u Q = kf Q - xq, xq = xr Q = iq + phi
                float xq = xr * (float)A.lutQ;
                float fiq = floorf(xq);
                float phi = xq - fiq;
                int iq1 = (int)fiq + 1;
                int php = iq1 & (A.lutQ - 1);           // (iq+1) mod Q (Q power of 2)
                int aa = (iq1 - php) / A.lutQ;          // floor((iq+1)/Q)
                int ph = (A.lutQ - php) & (A.lutQ - 1);
                int jsh = aa + (php > 0 ? 1 : 0);
                int rowbase = ph * A.lut_cols + A.lut_joff - jsh;
                rec = make_float2(__int_as_float(rowbase), phi);
                recA = amp;
              } else if (MODE == 3) {  // texture LUT: coordinate offset, amplitude
                rec = make_float2(fmaf(-xr, A.texQ, A.tex_off), amp);
              } else {
                // hoisted sinc numerator: sin(pi u) = -(-1)^(kf - j) sin(pi f), u = kf - xr, xr = j + f
                float fj = floorf(xr);
                float f = xr - fj;
                if (f == 0.f) {  // exact integer delay: nudge by one ulp (reading R3)
                  xr = nextafterf(xr, 1e30f);
                  fj = floorf(xr);
                  f = xr - fj;
                }
                const int jj = (int)fj;
                float cc = -amp * sinpi01(f) * 0.318309886183790672f;
                if (jj & 1) cc = -cc;
                if (MODE == 0) rec = make_float2(-xr * A.invHs, cc * A.invHs);
                else rec = make_float2(-xr * (0.5f * A.invHs), cc * (0.5f * A.invHs) * 1024.f);
              }
            }
          }
          const int dst = filled + (gi - base);
          sm.rec[dst] = rec;
          if (MODE == 1) sm.recA[dst] = recA;
          sm.bin[dst] = b;
        }
      }
      filled += take;
      base += take;
      if (filled == kCap) {
        __syncthreads();
        process_window(filled);
        filled = 0;
      }
    }
    __syncthreads();  // column records are replaced by the next batch
  }
  if (filled > 0) {
    __syncthreads();
    process_window(filled);
  }

  // ---- reduce lane groups, apply the lane sign, write the tile ----------------
#pragma unroll
  for (int s = 0; s < kSubPerWarp; s++) {
    float a = acc[s].x + acc[s].y;
    a += __shfl_xor_sync(0xffffffffu, a, 8);
    a += __shfl_xor_sync(0xffffffffu, a, 16);
    if (MODE == 0) { if (kfs[s] & 1) a = -a; }
    else if (MODE == 2) { a *= (1.f / 1024.f); if (kfs[s] & 1) a = -a; }
    if (grp == 0) sm.outtile[(s * kWarps + warp) * kS + li] = a;
  }
  if (P > 1) {
    cluster.sync();
    if (prank == 0 && tid < kTC) {
      float s = sm.outtile[tid];
      for (int r = 1; r < P; r++) s += cluster.map_shared_rank(&sm.outtile[0], r)[tid];
      sm.outtile[tid] = s;
    }
    cluster.sync();
  } else {
    __syncthreads();
  }
  if (prank == 0 && tid < T.te - T.t0) A.out[T.row + T.t0 + tid] = sm.outtile[tid];
}

// ----------------------------------------------------------------------------
// image-parameter hook (gpurir_image_params): one thread per lattice image
// ----------------------------------------------------------------------------
__global__ void image_params_kernel(IsmArgs A, double* x_out, float* A_out) {
  __shared__ RirGeom g;
  if (threadIdx.x == 0) load_geom(A, 0, g, A.status);
  __syncthreads();
  int Nx = g.nhi[0] - g.nlo[0], Ny = g.nhi[1] - g.nlo[1], Nz = g.nhi[2] - g.nlo[2];
  long long N = (long long)Nx * Ny * Nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    int nx = g.nlo[0] + (int)(i % Nx), ny = g.nlo[1] + (int)((i / Nx) % Ny), nz = g.nlo[2] + (int)(i / ((long long)Nx * Ny));
    double dx = image_coord(nx, g.L[0], g.s[0]) - g.r[0];
    double dy = image_coord(ny, g.L[1], g.s[1]) - g.r[1];
    double dz = image_coord(nz, g.L[2], g.s[2]) - g.r[2];
    double x2 = fma(dz, dz, dx * dx + dy * dy) * (A.fs_over_c * A.fs_over_c);
    if (x2 == 0.0) { atomicOr(A.status, kStatusDegenerate); x_out[i] = 0.0; A_out[i] = 0.f; continue; }
    float x0f;
    (void)delay_rel(x2, 0, x0f);
    double x0d = (double)x0f;
    double xfull = x0d + (x2 - x0d * x0d) / (2.0 * x0d);  // same fp64 Newton step, reference 0
    const float rx = rcp_approx(x0f);
    uint32_t sgn = 0; bool zero = false;
    float lb = axis_beta(nx, 0, g, sgn, zero) + axis_beta(ny, 1, g, sgn, zero) + axis_beta(nz, 2, g, sgn, zero);
    float bn = zero ? 0.f : ex2_approx(lb);
    if (sgn) bn = -bn;
    float cth = ((float)dx * g.o[0] + (float)dy * g.o[1] + (float)dz * g.o[2]) * ((float)A.fs_over_c * rx);
    float gain = (g.a + (1.f - g.a) * cth) *
                 src_gain(src_col_dot(nx, ny, (float)dx, (float)dy, g), nz & 1, (float)dz, (float)A.fs_over_c * rx, g);
    x_out[i] = xfull;
    A_out[i] = bn * gain * rx * (float)A.fs_over_c * 0.0795774715459476679f;
  }
}

size_t ism_smem_bytes(int mode, int lut_rows, int lut_cols) {
  size_t s = sizeof(Smem);
  if (mode == 1) s += (size_t)lut_rows * lut_cols * sizeof(float2);
  return s;
}

template <int MODE>
static cudaError_t launch_mode(const cudaLaunchConfig_t& cfg, const IsmArgs& A) {
  cudaError_t e = cudaFuncSetAttribute(ism_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)cfg.dynamicSmemBytes);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, ism_kernel<MODE>, A);
}

cudaError_t launch_ism(const IsmArgs& A, int mode, int split, long long nclusters, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nclusters * split), 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = ism_smem_bytes(mode, A.lut_rows, A.lut_cols);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = split;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (mode) {
    case 0: return launch_mode<0>(cfg, A);
    case 1: return launch_mode<1>(cfg, A);
    case 3: return launch_mode<3>(cfg, A);
    default: return launch_mode<2>(cfg, A);
  }
}

cudaError_t launch_image_params(const IsmArgs& A, double* x_out, float* A_out, long long N, cudaStream_t stream) {
  long long nb = (N + 255) / 256;
  int blocks = (int)(nb < 148LL * 16 ? nb : 148LL * 16);
  if (blocks < 1) blocks = 1;
  image_params_kernel<<<blocks, 256, 0, stream>>>(A, x_out, A_out);
  return cudaGetLastError();
}

}  // namespace gpurir

// ism_common.cuh — device helpers shared by the ISM kernels (ism_kernel.cu, ism_ws_kernel.cu).
#pragma once

#include <cuda_fp16.h>

#include "device_common.cuh"
#include "kernels.h"

namespace gpurir {

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// sin(pi f) for f in [0, 1) with ~2e-7 relative accuracy (also near f = 0 and f = 1):
// h = min(f, 1 - f) (exact), sin(pi h) = h P(h^2), minimax degree 4.
__device__ __forceinline__ float sinpi01(float f) {
  float h = fminf(f, 1.f - f);
  float y = h * h;
  float p = fmaf(0.07768171280622482f, y, -0.5983065366744995f);
  p = fmaf(p, y, 2.5500807762145996f);
  p = fmaf(p, y, -5.167710304260254f);
  p = fmaf(p, y, 3.1415927410125732f);
  return h * p;
}

// ----------------------------------------------------------------------------
// Per-RIR geometry (single-room call or batch job)
// ----------------------------------------------------------------------------
__device__ __forceinline__ float pattern_const(int pattern) {  // C4
  return pattern == 0 ? 1.f : pattern == 1 ? 0.75f : pattern == 2 ? 0.5f : pattern == 3 ? 0.25f : 0.f;
}
// unit orientation of a directional pattern (0 for omni); a zero vector raises the status word
__device__ __forceinline__ void unit_orient(const float* v, int pattern, float* o, int* status) {
  float o0 = v[0], o1 = v[1], o2 = v[2];
  float on2 = o0 * o0 + o1 * o1 + o2 * o2;
  if (pattern != 0 && !(on2 > 0.f)) { atomicOr(status, kStatusZeroOrient); on2 = 1.f; }
  const float inv = pattern != 0 ? rsqrtf(on2) : 0.f;
  o[0] = o0 * inv; o[1] = o1 * inv; o[2] = o2 * inv;
}
static __device__ void geom_from(const float* L, const float* src, const float* rcv, const float* orv, const int* nb,
                                 int pattern, const float* ors, int spkr_pattern, const float* lb, unsigned neg,
                                 unsigned zero, RirGeom& g, int* status) {
  g.a = pattern_const(pattern);
  unit_orient(orv, pattern, g.o, status);
  g.as = pattern_const(spkr_pattern);  // source directivity (f3, reading R10)
  unit_orient(ors, spkr_pattern, g.os, status);
  for (int i = 0; i < 3; i++) {
    g.L[i] = L[i]; g.s[i] = src[i]; g.r[i] = rcv[i];
    g.nlo[i] = -(nb[i] / 2);          // ceil(-N/2)
    g.nhi[i] = (nb[i] + 1) / 2;       // ceil(N/2)
  }
  g.neg = neg; g.zero = zero;
  for (int w = 0; w < 6; w++) g.lb[w] = lb[w];
}

// Per-RIR geometry (single-room call or batch job) read straight from global memory.
static __device__ void load_geom(const IsmArgs& A, int m, RirGeom& g, int* status) {
  if (A.jobs) {
    const BatchJob& J = A.jobs[m];
    geom_from(J.L, J.src, J.rcv, J.orv, J.nb, J.pattern, J.ors, J.spkr_pattern, J.lb, J.neg, J.zero, g, status);
  } else {
    int ms = m / A.M_rcv, mr = m % A.M_rcv;
    const float zero3[3] = {0.f, 0.f, 0.f};
    geom_from(A.L, A.pos_src + 3 * ms, A.pos_rcv + 3 * mr, A.orv ? A.orv + 3 * mr : zero3, A.nb, A.pattern,
              A.ors ? A.ors + 3 * ms : zero3, A.spkr_pattern, A.lb, A.neg, A.zero, g, status);
  }
}

// Source directivity (f3, reading R10): image n radiates along p_r - p_n with the source orientation mirrored on
// the axes where n is odd.  Column part (x, y) of cos(theta_s) * d: -(sx dx os_x + sy dy os_y), s = (-1)^n,
// d = p_n - p_r; the z part is added per image by src_gain.
__device__ __forceinline__ float src_col_dot(int nx, int ny, float dx, float dy, const RirGeom& g) {
  const float ox = (nx & 1) ? -g.os[0] : g.os[0], oy = (ny & 1) ? -g.os[1] : g.os[1];
  return -fmaf(dy, oy, dx * ox);
}
// g_s = as + (1 - as) cos(theta_s); inv_d = 1 / d.  Exactly 1 for an omni source (as = 1, os = 0).
__device__ __forceinline__ float src_gain(float sdot, int nz_odd, float dz, float inv_d, const RirGeom& g) {
  const float oz = nz_odd ? -g.os[2] : g.os[2];
  return fmaf(1.f - g.as, fmaf(-dz, oz, sdot) * inv_d, g.as);
}

// Exact n_z range of one side of a column: all n with lo <= Delta_z(n) <= hi, where
// Delta_z(n) = z_n - z_r is strictly increasing in n (image n lies in cell [nL, (n+1)L]).
__device__ __forceinline__ void z_range(const RirGeom& g, double invLz, double lo, double hi, int& first,
                                        int& last) {
  const double Lz = g.L[2], sz = g.s[2], rz = g.r[2];
  int a = (int)floor((rz + lo) * invLz);
  if (image_coord(a, Lz, sz) - rz < lo) a++;
  int b = (int)floor((rz + hi) * invLz);
  if (image_coord(b, Lz, sz) - rz > hi) b--;
  first = a;
  last = b;
}


// Eqs. 5-6 for one lane over record pairs pp[0], pp[kG], ... < pend (see ism_kernel.cu for the derivation):
// acc += C' w(u) / v, v = (k - x)/Hs, sigma = v^2 - rho^2 clamped <= 0, w = (sigma p(sigma))^2.
struct TapConst {
  float2 kv2, a3, a2, a1, a0;
  float up;
};
// Eq. 5-6 per pair of records: acc += C' w(v) / v with v = (k - x)/Hs.  The window is c(u)^2 where
// u = min(max(v^2 + 1 - rho^2, 0), 1) (one FFMA.SAT per record: u = 1 at and beyond the window edge,
// where c(1) = 0 exactly) and c is the degree-3 polynomial of fill_common (R5).
__device__ __forceinline__ TapConst make_tap_const(const IsmArgs& A, float kv) {
  TapConst K;
  K.kv2 = make_float2(kv, kv);
  K.a3 = make_float2(A.wa[3], A.wa[3]);
  K.a2 = make_float2(A.wa[2], A.wa[2]); K.a1 = make_float2(A.wa[1], A.wa[1]);
  K.a0 = make_float2(A.wa[0], A.wa[0]);
  K.up = A.urho;
  return K;
}
__device__ __forceinline__ float2 tap_pair(const float4 p, const TapConst& K, float2 a2) {
  const float2 v = __fadd2_rn(K.kv2, make_float2(p.x, p.y));
  const float2 u = make_float2(__saturatef(fmaf(v.x, v.x, K.up)), __saturatef(fmaf(v.y, v.y, K.up)));
  float2 c = __ffma2_rn(K.a3, u, K.a2);
  c = __ffma2_rn(c, u, K.a1);
  c = __ffma2_rn(c, u, K.a0);
  const float2 w = __fmul2_rn(c, c);
  const float2 r = make_float2(rcp_approx(v.x), rcp_approx(v.y));
  return __ffma2_rn(make_float2(p.z, p.w), __fmul2_rn(w, r), a2);
}
__device__ __forceinline__ float2 tap_loop(const float4* pp, const float4* pend, const TapConst& K, float2 a2) {
#ifdef GPURIR_EXPERIMENT_SKIP_TAPS  // profiling experiment only: producer-bound time
  if (pend - pp < 1000000) return a2;
#endif
  float2 a3 = make_float2(0.f, 0.f);  // second accumulator: two independent FFMA2 chains
  for (; pp + 3 * kG < pend; pp += 4 * kG) {
    const float4 p0 = pp[0], p1 = pp[kG], p2 = pp[2 * kG], p3 = pp[3 * kG];
    a2 = tap_pair(p0, K, a2);
    a3 = tap_pair(p1, K, a3);
    a2 = tap_pair(p2, K, a2);
    a3 = tap_pair(p3, K, a3);
  }
  for (; pp < pend; pp += kG) a2 = tap_pair(pp[0], K, a2);
  a2.x += a3.x;
  a2.y += a3.y;
  return a2;
}

// fp16 / half2 mode: t - tau in fp32, Hann window by the Eq. 11 polynomial cos(pi x)
// at x = u / (2H) (reading C12) in half2 Horner (Eq. 12), the bounded product C/x in fp32 -> half2,
// half2 partial sums flushed to fp32 every 4 unrolled iterations (reading C13).
struct TapConstH {
  float2 kx2;
  __half2 c6, c4, c2, c0, xcl;
};
__device__ __forceinline__ __half2 tap_pair_h(const float4 p, const TapConstH& K, __half2 acch) {
  const float2 x = __fadd2_rn(K.kx2, make_float2(p.x, p.y));  // x' = (k - tau fs) / (2 Hs), fp32
  const __half2 hx = __float22half2_rn(x);
  const __half2 x2 = __hmin2(__hmul2(hx, hx), K.xcl);         // clamp at the window edge |u/(2H)| = 1/2
  __half2 q = __hfma2(K.c6, x2, K.c4);
  q = __hfma2(q, x2, K.c2);
  q = __hfma2(q, x2, K.c0);                                    // cos(pi x), Eq. 11
  const __half2 w = __hmul2(q, q);                             // Hann window
  const float2 r = make_float2(rcp_approx(x.x), rcp_approx(x.y));
  const float2 cq = __fmul2_rn(make_float2(p.z, p.w), r);     // bounded by ~A (scaled 2^10)
  return __hfma2(w, __float22half2_rn(cq), acch);
}
__device__ __forceinline__ float2 tap_loop_h(const float4* pp, const float4* pend, const TapConstH& K, float2 a2) {
  const __half2 z = __float2half2_rn(0.f);
  int it = 0;
  __half2 h0 = z, h1 = z;
  for (; pp + 3 * kG < pend; pp += 4 * kG) {
    const float4 p0 = pp[0], p1 = pp[kG], p2 = pp[2 * kG], p3 = pp[3 * kG];
    h0 = tap_pair_h(p0, K, h0);
    h1 = tap_pair_h(p1, K, h1);
    h0 = tap_pair_h(p2, K, h0);
    h1 = tap_pair_h(p3, K, h1);
    if (++it == 4) {  // at most 8 half2 products per partial sum
      const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
      a2.x += f0.x + f1.x; a2.y += f0.y + f1.y;
      h0 = z; h1 = z; it = 0;
    }
  }
  for (; pp < pend; pp += kG) h0 = tap_pair_h(pp[0], K, h0);
  const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
  a2.x += f0.x + f1.x; a2.y += f0.y + f1.y;
  return a2;
}

// Texture-LUT mode (the paper's own LUT design): record pairs (q_e, q_o, A_e, A_o) with
// q = tex_off - x Q (x relative to the tile centre); per tap coordinate = kq + q (kq = k Q), the texture unit
// interpolates T linearly (8-bit fractional weight) and returns 0 outside the table (border addressing).
__device__ __forceinline__ float2 tap_pair_tex(const float4 p, cudaTextureObject_t tex, float2 kq2, float2 a2) {
  const float2 q = __fadd2_rn(kq2, make_float2(p.x, p.y));
  const float2 t = make_float2(tex1D<float>(tex, q.x), tex1D<float>(tex, q.y));
  return __ffma2_rn(make_float2(p.z, p.w), t, a2);
}
__device__ __forceinline__ float2 tap_loop_tex(const float4* pp, const float4* pend, cudaTextureObject_t tex, float kq,
                                               float2 a2) {
  const float2 kq2 = make_float2(kq, kq);
  float2 a3 = make_float2(0.f, 0.f);
  for (; pp + 3 * kG < pend; pp += 4 * kG) {
    const float4 p0 = pp[0], p1 = pp[kG], p2 = pp[2 * kG], p3 = pp[3 * kG];
    a2 = tap_pair_tex(p0, tex, kq2, a2);
    a3 = tap_pair_tex(p1, tex, kq2, a3);
    a2 = tap_pair_tex(p2, tex, kq2, a2);
    a3 = tap_pair_tex(p3, tex, kq2, a3);
  }
  for (; pp < pend; pp += kG) a2 = tap_pair_tex(pp[0], tex, kq2, a2);
  a2.x += a3.x;
  a2.y += a3.y;
  return a2;
}

}  // namespace gpurir

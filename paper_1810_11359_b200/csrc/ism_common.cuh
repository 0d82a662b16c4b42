// ism_common.cuh — device helpers shared by the ISM kernels (ism_kernel.cu, ism_ws_kernel.cu).
#pragma once

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
static __device__ void load_geom(const IsmArgs& A, int m, RirGeom& g, int* status) {
  float L[3], beta[6], src[3], rcv[3], orv[3] = {0.f, 0.f, 0.f};
  int nb[3], pattern;
  if (A.jobs) {
    const BatchJob& J = A.jobs[m];
    for (int i = 0; i < 3; i++) { L[i] = J.L[i]; src[i] = J.src[i]; rcv[i] = J.rcv[i]; orv[i] = J.orv[i]; nb[i] = J.nb[i]; }
    for (int i = 0; i < 6; i++) beta[i] = J.beta[i];
    pattern = J.pattern;
  } else {
    int ms = m / A.M_rcv, mr = m % A.M_rcv;
    for (int i = 0; i < 3; i++) {
      L[i] = A.L[i]; nb[i] = A.nb[i];
      src[i] = A.pos_src[3 * ms + i];
      rcv[i] = A.pos_rcv[3 * mr + i];
      if (A.orv) orv[i] = A.orv[3 * mr + i];
    }
    for (int i = 0; i < 6; i++) beta[i] = A.beta[i];
    pattern = A.pattern;
  }
  g.a = pattern == 0 ? 1.f : pattern == 1 ? 0.75f : pattern == 2 ? 0.5f : pattern == 3 ? 0.25f : 0.f;  // C4
  float on = sqrtf(orv[0] * orv[0] + orv[1] * orv[1] + orv[2] * orv[2]);
  if (pattern != 0 && !(on > 0.f)) { atomicOr(status, kStatusZeroOrient); on = 1.f; }
  for (int i = 0; i < 3; i++) {
    g.L[i] = L[i]; g.s[i] = src[i]; g.r[i] = rcv[i];
    g.o[i] = pattern != 0 ? orv[i] / on : 0.f;
    g.nlo[i] = -(nb[i] / 2);          // ceil(-N/2)
    g.nhi[i] = (nb[i] + 1) / 2;       // ceil(N/2)
  }
  g.neg = 0; g.zero = 0;
  for (int w = 0; w < 6; w++) {
    float b = beta[w];
    if (b < 0.f) g.neg |= 1u << w;
    if (b == 0.f) { g.zero |= 1u << w; g.lb[w] = 0.f; }
    else g.lb[w] = log2f(fabsf(b));
  }
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


}  // namespace gpurir

/*
 * oracle.c — plain, slow, obviously-correct double-precision CPU oracle for
 * the Image Source Method RIR path of gpuRIR (arXiv 1810.11359).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * in paper_1810_11359_b200/ and never includes or links it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, with the equation or
 * section it falls in; "C<k>" = reading k of SURVEY.md §8(c), restated in
 * DESIGN.md §"Readings".
 *
 * Every function follows the paper's definition written out, in the paper's
 * order and notation; there is no blocking, fusion or reordering.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): beta = 0 direct path (closed
 * form), single-image renders (Eq. 6 closed forms), brute-force mirror
 * enumeration of the image set, reciprocity, lattice completeness, Sabine
 * helper values printed in SPEC.md, Philox4x32-10 known-answer vectors,
 * logistic-noise moments, energy-decay slope vs Sabine, the dense
 * formulation vs the support-restricted loop, cross-implementation goldens;
 * for the f3 extensions: source directivity vs the mirror BFS's reflected
 * orientation, vs the specular point of a first-order reflection, special
 * angles, directional reciprocity; weighted beta vs Sabine's Eq. (7).
 * Functions without such a pin: none (oracle_lut_build and the Eq. 10/11
 * polynomials are pinned by the values the paper prints for their
 * coefficients and by their closed-form special points).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL 1
#define OR_EDEGENERATE 2
#define OR_EINFEASIBLE 3

static const double OR_PI = 3.14159265358979323846264338327950288;

/* ------------------------------------------------------------------ */
/* Sample-count reading (C9): n = ceil(T*fs); a product within 1e-6 of */
/* an integer from above counts as that integer (binary rounding of the */
/* inputs must not add a sample).                                       */
/* ------------------------------------------------------------------ */
long oracle_nsamples(double T, double fs) {
  double p = T * fs;
  long n = (long)ceil(p - 1e-6);
  return n < 0 ? 0 : n;
}

/* ------------------------------------------------------------------ */
/* A1, P:90 (§2.1): grid N of image sources, ceil(-N/2) <= n < ceil(N/2) */
/* ------------------------------------------------------------------ */
static int lattice_lo(int N) { return (int)ceil(-N / 2.0); }
static int lattice_hi(int N) { return (int)ceil(N / 2.0); } /* exclusive */

/* A2, Eq. (1): image coordinate along one axis. */
double oracle_image_coord(int n, double L, double s) {
  if (n % 2 == 0) return n * L + s;
  return (n + 1) * L - s;
}

/* A4, P:109 + reading C2: crossings of wall 0 = |floor(n/2)|, wall 1 = |ceil(n/2)|. */
void oracle_wall_crossings(int n, int* c0, int* c1) {
  *c0 = abs((int)floor(n / 2.0));
  *c1 = abs((int)ceil(n / 2.0));
}

/* A16 + reading C4: first-order polar pattern g = a + (1-a) cos(theta). */
static double pattern_a(int pattern) {
  switch (pattern) {
    case 0: return 1.0;   /* omni */
    case 1: return 0.75;  /* subcardioid */
    case 2: return 0.5;   /* cardioid */
    case 3: return 0.25;  /* hypercardioid */
    case 4: return 0.0;   /* bidirectional */
  }
  return -1.0;
}

/* Source directivity (NEXT row f3, reading R10; not in the paper, which  */
/* gives only the receiver pattern): the image source n is the     */
/* source mirrored along every axis on which Eq. (1) mirrors it (n odd),  */
/* so it carries the source orientation o_s with those components negated */
/* and radiates toward the receiver along p_r - p_n:                      */
/* g_s = a_s + (1 - a_s) (M_n o_s) . (p_r - p_n) / d_n, M_n = diag((-1)^n). */
static double source_gain(double a_s, const double os[3], const int n[3], const double p[3], const double rcv[3],
                          double d) {
  double c = 0.0;
  for (int ax = 0; ax < 3; ax++) {
    double o = (n[ax] % 2 != 0) ? -os[ax] : os[ax];
    c += o * (rcv[ax] - p[ax]);
  }
  return a_s + (1.0 - a_s) * c / d;
}

/* Unit orientation of a directional pattern; EINVAL for a zero vector. */
static int unit_orientation(int pattern, const double* v, double o[3]) {
  o[0] = o[1] = o[2] = 0.0;
  if (pattern == 0) return OR_OK;
  if (!v) return OR_EINVAL;
  double on = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  if (!(on > 0.0)) return OR_EINVAL;
  for (int i = 0; i < 3; i++) o[i] = v[i] / on;
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Eq. (6), P:127-134 with T_w = window length (s), f_c = fs/2 (C7):   */
/* delta'(t) = 1/2 (1 + cos(2 pi t / T_w)) sinc(2 pi f_c t), |t|<T_w/2 */
/* Argument t in seconds.                                              */
/* ------------------------------------------------------------------ */
double oracle_windowed_sinc(double t, double Tw, double fc) {
  if (!(t > -Tw / 2.0 && t < Tw / 2.0)) return 0.0; /* C8: open support */
  double win = 0.5 * (1.0 + cos(2.0 * OR_PI * t / Tw));
  double arg = 2.0 * OR_PI * fc * t;
  double sinc = (arg == 0.0) ? 1.0 : sin(arg) / arg;
  return win * sinc;
}

/* ------------------------------------------------------------------ */
/* Eq. (7): Sabine T60 = 0.161 V / sum S_i alpha_i,         */
/* alpha_i = 1 - beta_i^2.  Wall order (x0,x1,y0,y1,z0,z1).     */
/* Returns +inf when every wall reflects perfectly.                    */
/* ------------------------------------------------------------------ */
double oracle_sabine_t60(const double room[3], const double beta[6]) {
  double V = room[0] * room[1] * room[2];
  double S[6] = {room[1] * room[2], room[1] * room[2], room[0] * room[2],
                 room[0] * room[2], room[0] * room[1], room[0] * room[1]};
  double den = 0.0;
  for (int i = 0; i < 6; i++) den += S[i] * (1.0 - beta[i] * beta[i]);
  if (den <= 0.0) return INFINITY;
  return 0.161 * V / den;
}

/* A17, P:276 + reading C17: uniform alpha = 0.161 V / (T60 S_total),   */
/* beta = sign * sqrt(1 - alpha).  alpha > 1 -> EINFEASIBLE unless clamp */
/* (then beta = 0, anechoic).  Returns status; *clamped set if clamped. */
int oracle_beta_sabine(const double room[3], double T60, int sign, int clamp, double beta_out[6],
                       int* clamped) {
  if (clamped) *clamped = 0;
  if (!(T60 > 0.0) || !(room[0] > 0 && room[1] > 0 && room[2] > 0)) return OR_EINVAL;
  double V = room[0] * room[1] * room[2];
  double Stot = 2.0 * (room[0] * room[1] + room[0] * room[2] + room[1] * room[2]);
  double alpha = 0.161 * V / (T60 * Stot);
  if (alpha > 1.0) {
    if (!clamp) return OR_EINFEASIBLE;
    if (clamped) *clamped = 1;
    for (int i = 0; i < 6; i++) beta_out[i] = 0.0;
    return OR_OK;
  }
  double b = sqrt(1.0 - alpha) * (sign < 0 ? -1.0 : 1.0);
  for (int i = 0; i < 6; i++) beta_out[i] = b;
  return OR_OK;
}

/* NEXT row f3 (the helper of P:276 with non-uniform walls, reading R9): */
/* alpha_i = w_i alpha0 with alpha0 fixed by Eq. (7), 0.161 V / sum_i S_i w_i alpha0   */
/* = T60, i.e. alpha0 = 0.161 V / (T60 sum_i S_i w_i); beta_i = sign sqrt(1 - alpha_i). */
/* Weights w_i >= 0, not all zero.  Some alpha_i > 1 -> EINFEASIBLE unless clamp (then  */
/* beta = 0 everywhere, anechoic).                                                     */
int oracle_beta_sabine_weighted(const double room[3], double T60, const double w[6], int sign, int clamp,
                                double beta_out[6], int* clamped) {
  if (clamped) *clamped = 0;
  if (!(T60 > 0.0) || !(room[0] > 0 && room[1] > 0 && room[2] > 0)) return OR_EINVAL;
  double V = room[0] * room[1] * room[2];
  double S[6] = {room[1] * room[2], room[1] * room[2], room[0] * room[2],
                 room[0] * room[2], room[0] * room[1], room[0] * room[1]};
  double Sw = 0.0;
  for (int i = 0; i < 6; i++) {
    if (!(w[i] >= 0.0)) return OR_EINVAL;
    Sw += S[i] * w[i];
  }
  if (!(Sw > 0.0)) return OR_EINVAL;
  double alpha0 = 0.161 * V / (T60 * Sw);
  for (int i = 0; i < 6; i++) {
    if (w[i] * alpha0 > 1.0) {
      if (!clamp) return OR_EINFEASIBLE;
      if (clamped) *clamped = 1;
      for (int j = 0; j < 6; j++) beta_out[j] = 0.0;
      return OR_OK;
    }
  }
  for (int i = 0; i < 6; i++) beta_out[i] = sqrt(1.0 - w[i] * alpha0) * (sign < 0 ? -1.0 : 1.0);
  return OR_OK;
}

/* A18: time to reach an attenuation of att_dB on the exponential */
/* decay whose 60 dB time is T60: t = att/60 * T60.             */
double oracle_att2t(double att_dB, double T60) { return att_dB / 60.0 * T60; }

/* A19, P:276 + reading C6: images per axis reaching time T without lost */
/* reflections: N = 2 (ceil(c T / L) + 1) + 1.                           */
int oracle_t2n(double T, const double room[3], double c, int nb_out[3]) {
  if (!(T > 0.0) || !(c > 0.0)) return OR_EINVAL;
  for (int a = 0; a < 3; a++) {
    if (!(room[a] > 0.0)) return OR_EINVAL;
    nb_out[a] = 2 * ((int)ceil(c * T / room[a]) + 1) + 1;
  }
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (reading C16; Salmon et al. 2011, the generator cuRAND */
/* exposes as curand_init(seed, subsequence, offset)).                 */
/* ------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; r++) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* C16: uniform draw for (seed, global RIR index r, sample k):            */
/* word (k & 3) of Philox(key = seed, ctr = (lo(k>>2), hi(k>>2), lo(r),   */
/* hi(r))), mapped to u = (2 (w >> 9) + 1) 2^-24 in (0, 1).               */
double oracle_uniform(uint64_t seed, uint64_t r, uint64_t k) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint64_t q = k >> 2;
  uint32_t ctr[4] = {(uint32_t)q, (uint32_t)(q >> 32), (uint32_t)r, (uint32_t)(r >> 32)};
  uint32_t out[4];
  oracle_philox4x32_10(ctr, key, out);
  uint32_t w = out[k & 3];
  return (2.0 * (double)(w >> 9) + 1.0) / 16777216.0;
}

/* unit-variance logistic noise (reading C16):            */
/* x = (sqrt(3)/pi) ln(u / (1 - u)).                                    */
double oracle_logistic(double u) { return sqrt(3.0) / OR_PI * log(u / (1.0 - u)); }

/* ------------------------------------------------------------------ */
/* Image set of one source/receiver pair (Table 2 calcAmpTau, Eqs. 2-4 */
/* P:99-113, A16).  Lattice order: n_x fastest, then n_y, then n_z.    */
/* Outputs (each optional): n_out[3*i], x_out[i] = tau_n * fs (delay   */
/* in samples), A_out[i] = beta_n g / (4 pi d_n), beta_out[i] = beta_n. */
/* Returns the number of images, or -status on error.                  */
/* ------------------------------------------------------------------ */
long oracle_image_set(const double room[3], const double beta[6], const double src[3], const double rcv[3],
                      const double orv[3], int pattern, const double ors[3], int spkr_pattern, const int nb[3],
                      double fs, double c, int* n_out, double* x_out, double* A_out, double* beta_out) {
  double a = pattern_a(pattern), a_s = pattern_a(spkr_pattern);
  if (a < 0.0 || a_s < 0.0) return -OR_EINVAL;
  double o[3], os[3];
  if (unit_orientation(pattern, orv, o) != OR_OK) return -OR_EINVAL;
  if (unit_orientation(spkr_pattern, ors, os) != OR_OK) return -OR_EINVAL;
  long idx = 0;
  for (int nz = lattice_lo(nb[2]); nz < lattice_hi(nb[2]); nz++) {
    for (int ny = lattice_lo(nb[1]); ny < lattice_hi(nb[1]); ny++) {
      for (int nx = lattice_lo(nb[0]); nx < lattice_hi(nb[0]); nx++) {
        int n[3] = {nx, ny, nz};
        double p[3], bn = 1.0;
        for (int ax = 0; ax < 3; ax++) {
          p[ax] = oracle_image_coord(n[ax], room[ax], src[ax]); /* Eq. (1) */
          int c0, c1;
          oracle_wall_crossings(n[ax], &c0, &c1);
          bn *= pow(beta[2 * ax], c0) * pow(beta[2 * ax + 1], c1);
        }
        /* Eq. (2) with the image position p_n (erratum C1). */
        double D[3] = {p[0] - rcv[0], p[1] - rcv[1], p[2] - rcv[2]};
        double d = sqrt(D[0] * D[0] + D[1] * D[1] + D[2] * D[2]);
        if (d == 0.0) return -OR_EDEGENERATE;
        double g = 1.0;
        if (pattern != 0) g = a + (1.0 - a) * (D[0] * o[0] + D[1] * o[1] + D[2] * o[2]) / d;
        if (spkr_pattern != 0) g *= source_gain(a_s, os, n, p, rcv, d);
        if (n_out) { n_out[3 * idx] = nx; n_out[3 * idx + 1] = ny; n_out[3 * idx + 2] = nz; }
        if (x_out) x_out[idx] = d / c * fs;                   /* Eq. (3): tau = d / c */
        if (A_out) A_out[idx] = bn * g / (4.0 * OR_PI * d);   /* Eq. (4), g = receiver x source gain */
        if (beta_out) beta_out[idx] = bn;
        idx++;
      }
    }
  }
  return idx;
}

/* ------------------------------------------------------------------ */
/* One RIR: Eq. (5) with delta' of Eq. (6) for 0 <= k < nISM, then the  */
/* diffuse tail (readings C14, C15, C16) for          */
/* nISM <= k < nSamples.  h must hold nSamples doubles.                 */
/* dense = 1 evaluates delta'(k - x) for every k of every image (the    */
/* paper's generateRIR formulation); dense = 0 visits only the   */
/* support |k - x| < T_w fs / 2 (identical).                     */
/* ------------------------------------------------------------------ */
static int one_rir(const double room[3], const double beta[6], const double src[3], const double rcv[3],
                   const double* orv, int pattern, const double* ors, int spkr_pattern, const int nb[3], long nISM,
                   long nS, double fs, double c, double Tw, uint64_t seed, uint64_t r_global, int dense, double* h) {
  for (long k = 0; k < nS; k++) h[k] = 0.0;
  double a = pattern_a(pattern), a_s = pattern_a(spkr_pattern);
  if (a < 0.0 || a_s < 0.0) return OR_EINVAL;
  double o[3], os[3];
  if (unit_orientation(pattern, orv, o) != OR_OK) return OR_EINVAL;
  if (unit_orientation(spkr_pattern, ors, os) != OR_OK) return OR_EINVAL;
  double H = Tw * fs / 2.0; /* half window in samples */
  long nI = nISM < nS ? nISM : nS;
  for (int nz = lattice_lo(nb[2]); nz < lattice_hi(nb[2]); nz++) {
    for (int ny = lattice_lo(nb[1]); ny < lattice_hi(nb[1]); ny++) {
      for (int nx = lattice_lo(nb[0]); nx < lattice_hi(nb[0]); nx++) {
        int n[3] = {nx, ny, nz};
        double p[3], bn = 1.0;
        for (int ax = 0; ax < 3; ax++) {
          p[ax] = oracle_image_coord(n[ax], room[ax], src[ax]);
          int c0, c1;
          oracle_wall_crossings(n[ax], &c0, &c1);
          bn *= pow(beta[2 * ax], c0) * pow(beta[2 * ax + 1], c1);
        }
        double D[3] = {p[0] - rcv[0], p[1] - rcv[1], p[2] - rcv[2]};
        double d = sqrt(D[0] * D[0] + D[1] * D[1] + D[2] * D[2]);
        if (d == 0.0) return OR_EDEGENERATE;
        double g = 1.0;
        if (pattern != 0) g = a + (1.0 - a) * (D[0] * o[0] + D[1] * o[1] + D[2] * o[2]) / d;
        if (spkr_pattern != 0) g *= source_gain(a_s, os, n, p, rcv, d);
        double A = bn * g / (4.0 * OR_PI * d);
        double tau = d / c;
        if (dense) {
          for (long k = 0; k < nI; k++) h[k] += A * oracle_windowed_sinc(k / fs - tau, Tw, fs / 2.0);
        } else {
          double x = tau * fs;
          long klo = (long)floor(x - H) + 1;
          long khi = (long)ceil(x + H) - 1;
          if (klo < 0) klo = 0;
          if (khi > nI - 1) khi = nI - 1;
          for (long k = klo; k <= khi; k++) h[k] += A * oracle_windowed_sinc(k / fs - tau, Tw, fs / 2.0);
        }
      }
    }
  }
  if (nI < nS) {
    /* Envelope prediction (envPred): Sabine T60 (Eq. 7), power     */
    /* envelope P(t) = A_env exp(-kappa t), kappa = 6 ln 10 / T60 (Eq. 8,  */
    /* reading C14).  A_env from the last 10 ms of ISM before Tdiff,       */
    /* clipped at the direct-path sample, by exact averaging (C15).        */
    double T60 = oracle_sabine_t60(room, beta);
    double kappa = isinf(T60) ? 0.0 : 6.0 * log(10.0) / T60;
    double Dd[3] = {src[0] - rcv[0], src[1] - rcv[1], src[2] - rcv[2]};
    double x_dp = sqrt(Dd[0] * Dd[0] + Dd[1] * Dd[1] + Dd[2] * Dd[2]) / c * fs;
    long w0 = nI - (long)llround(0.010 * fs);
    long wdp = (long)ceil(x_dp);
    if (wdp > w0) w0 = wdp;
    if (w0 < 0) w0 = 0;
    double Aenv = 0.0;
    if (w0 < nI) {
      double sh = 0.0, se = 0.0;
      for (long k = w0; k < nI; k++) {
        sh += h[k] * h[k];
        se += exp(-kappa * k / fs);
      }
      long nw = nI - w0;
      Aenv = (sh / nw) / (se / nw);
    }
    /* diffRev: logistic noise times sqrt(P(t)). */
    for (long k = nI; k < nS; k++) {
      double u = oracle_uniform(seed, r_global, (uint64_t)k);
      h[k] = sqrt(Aenv * exp(-kappa * k / fs)) * oracle_logistic(u);
    }
  }
  return OR_OK;
}

/* Full call: RIR r = m_src * M_rcv + m_rcv, output [M_src][M_rcv][nSamples]. */
/* src: M_src x 3, rcv: M_rcv x 3, orv: M_rcv x 3 or NULL (omni receivers),          */
/* ors: M_src x 3 or NULL (omni sources, reading R10).                                */
int oracle_simulate_rir(const double room[3], const double beta[6], const double* src, int M_src,
                        const double* rcv, int M_rcv, const double* orv, int pattern, const double* ors,
                        int spkr_pattern, const int nb[3],
                        double Tdiff, double Tmax, double fs, double c, double Tw, uint64_t seed,
                        uint64_t rir_index_base, int dense, int nthreads, double* out) {
  if (M_src <= 0 || M_rcv <= 0 || !(fs > 0) || !(c > 0) || !(Tmax > 0) || Tdiff < 0) return OR_EINVAL;
  if (nb[0] < 1 || nb[1] < 1 || nb[2] < 1) return OR_EINVAL;
  for (int i = 0; i < 6; i++)
    if (fabs(beta[i]) > 1.0) return OR_EINVAL;
  if (pattern < 0 || pattern > 4) return OR_EINVAL;
  if (pattern != 0 && !orv) return OR_EINVAL;
  if (spkr_pattern < 0 || spkr_pattern > 4) return OR_EINVAL;
  if (spkr_pattern != 0 && !ors) return OR_EINVAL;
  long nS = oracle_nsamples(Tmax, fs);
  long nISM = oracle_nsamples(Tdiff, fs);
  int M = M_src * M_rcv;
  int status = OR_OK;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int r = 0; r < M; r++) {
    int ms = r / M_rcv, mr = r % M_rcv;
    int st = one_rir(room, beta, src + 3 * ms, rcv + 3 * mr, orv ? orv + 3 * mr : NULL, pattern,
                     ors ? ors + 3 * ms : NULL, spkr_pattern, nb, nISM, nS, fs, c, Tw, seed,
                     rir_index_base + (uint64_t)r, dense, out + (size_t)r * nS);
    if (st != OR_OK) {
#ifdef _OPENMP
#pragma omp critical
#endif
      status = st;
    }
  }
  return status;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ */
/* Eq. (9), with the window argument read as               */
/* 2 pi n / (Q fs T_w) (erratum C11): LUT[n] = delta'(n / (Q fs)) for  */
/* n in {-T_w Q fs / 2, ..., T_w Q fs / 2} (range rounded up).  */
/* Writes 2*half+1 entries (index 0 <-> n = -half); returns half.      */
/* ------------------------------------------------------------------ */
long oracle_lut_build(double Tw, double fs, int Q, double* out, long cap) {
  long half = (long)ceil(Tw * Q * fs / 2.0 - 1e-9);
  if (out) {
    if (2 * half + 1 > cap) return -1;
    for (long n = -half; n <= half; n++) {
      double win = 0.5 * (1.0 + cos(2.0 * OR_PI * n / (Q * fs * Tw)));
      double arg = OR_PI * n / Q;
      double sinc = (n == 0) ? 1.0 : sin(arg) / arg;
      double v = win * sinc;
      if (!((double)n / (Q * fs) > -Tw / 2.0 && (double)n / (Q * fs) < Tw / 2.0)) v = 0.0; /* C8 */
      out[n + half] = v;
    }
  }
  return half;
}

/* LUT read-out: linear interpolation between the closest entries */
/* at fractional index t Q fs; 0 outside the table.               */
double oracle_lut_lookup(const double* lut, long half, int Q, double fs, double t) {
  double pos = t * Q * fs;
  double i0 = floor(pos);
  double w = pos - i0;
  long j = (long)i0;
  if (j < -half || j + 1 > half) return 0.0;
  return lut[j + half] * (1.0 - w) + lut[j + 1 + half] * w;
}

/* Eq. (10): sin(pi x) ~ 2.326171875 x^5 - 5.14453125 x^3 + 3.140625 x on */
/* [-1/2, 1/2] after reducing x to that range; result negated in the 2nd/3rd quadrant. */
/* Horner form (Eq. 12) in x^2.                                          */
double oracle_sin_pi_poly(double x) {
  double k = nearbyint(x); /* x = k + y, y in [-1/2, 1/2] */
  double y = x - k;
  double y2 = y * y;
  double p = ((2.326171875 * y2 - 5.14453125) * y2 + 3.140625) * y;
  long ki = (long)k;
  return (ki % 2 == 0) ? p : -p; /* sin(pi (k + y)) = (-1)^k sin(pi y) */
}

/* Eq. (11): cos(pi x) ~ -1.2294921875 x^6 + 4.04296875 x^4 - 4.93359375 x^2 + 1 */
/* on [-1/2, 1/2], no reduction (reading C12).                                          */
double oracle_cos_pi_poly(double x) {
  double x2 = x * x;
  return ((-1.2294921875 * x2 + 4.04296875) * x2 - 4.93359375) * x2 + 1.0;
}

/* Convenience for the statistical pins: out[i] = logistic(uniform(seed, r, k0 + i)). */
void oracle_logistic_stream(uint64_t seed, uint64_t r, uint64_t k0, long n, double* out) {
  for (long i = 0; i < n; i++) out[i] = oracle_logistic(oracle_uniform(seed, r, k0 + (uint64_t)i));
}

/* ------------------------------------------------------------------ */
/* NEXT row f1 (§3.4): a moving */
/* source recorded by a microphone array.  The source signal is split  */
/* into n_points contiguous segments of floor(n_sig / n_points) samples */
/* (the last takes the remainder; reading R7 = SPEC S:414); segment p   */
/* is filtered by the RIRs of trajectory point p and the filtered       */
/* segments are overlap-added at their offsets:                 */
/*   out[m][t] = sum_j sig[j] rir[p(j)][m][t - j], 0 <= t - j < L,      */
/*   0 <= t < n_sig + L - 1.  rirs: [n_points][n_mics][L].              */
/* Direct time-domain convolution in double (the plain definition).    */
/* ------------------------------------------------------------------ */
int oracle_simulate_trajectory(const double* sig, long n_sig, const double* rirs, int n_points, int n_mics,
                               long L, double* out) {
  if (n_sig <= 0 || n_points <= 0 || n_mics <= 0 || L <= 0 || n_sig < n_points) return OR_EINVAL;
  long seglen = n_sig / n_points;
  long n_out = n_sig + L - 1;
  for (long i = 0; i < (long)n_mics * n_out; i++) out[i] = 0.0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int m = 0; m < n_mics; m++) {  /* microphones are independent (one thread each) */
    double* o = out + (size_t)m * n_out;
    for (long j = 0; j < n_sig; j++) {
      long p = j / seglen;
      if (p > n_points - 1) p = n_points - 1;
      const double* h = rirs + ((size_t)p * n_mics + m) * L;
      for (long tau = 0; tau < L; tau++) o[j + tau] += sig[j] * h[tau];
    }
  }
  return OR_OK;
}

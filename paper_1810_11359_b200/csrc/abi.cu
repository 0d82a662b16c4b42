// abi.cu — C ABI of libgpurir.so (include/gpurir.h): host-side validation,
// sizing (hot-path row a0 of SURVEY.md §8(a)), planning and launch sequence.
//
// Every step of the RIR path runs in the CUDA kernels of ism_kernel.cu and
// tail_kernel.cu; this file only validates, sizes and launches.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/gpurir.h"
#include "device_common.cuh"
#include "kernels.h"

using namespace gpurir;

namespace {

thread_local char g_cuda_err[256] = "";
constexpr unsigned kCounterRing = 256;

int cuda_fail(cudaError_t e, const char* where) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", where, cudaGetErrorString(e));
  return GPURIR_ECUDA;
}

// Per-device status word and LUT cache (lazily created, process lifetime).
struct LutEntry {  // one uploaded Eq. 9 table; entries are never overwritten (kernels may still read them)
  double Tw = 0, fs = 0;
  int Q = 0, rows = 0, cols = 0, joff = 0;
  float2* dev = nullptr;
};

struct TexEntry {  // one Eq. 9 table as a filtered 1-D texture (texture-LUT mode, f2); never destroyed
  double Tw = 0, fs = 0;
  int Q = 0;
  long long half = 0;
  cudaArray_t arr = nullptr;
  cudaTextureObject_t tex = 0;
};

struct PolyEntry {  // polyphase table of one (Tw, fs) (mode GPURIR_POLY, reading R11); never overwritten
  double Tw = 0, fs = 0;
  int ntaps = 0, mlo = 0;
  int nmi0 = 0, nn = 0;  // the rotated near channels' tap window (poly_fir_tables)
  float* dev = nullptr;
};

struct DeviceState {
  int* status = nullptr;
  std::vector<LutEntry> luts;
  std::vector<TexEntry> texs;
  std::vector<PolyEntry> polys;
  int* work_counter = nullptr;  // persistent-kernel work-queue heads, one per call in flight (ring)
  // gpurir_simulate_rir_host: copy stream, chunk events and a grow-only scratch buffer, owned by the device
  // state and used under host_mu (host calls on one device run one at a time)
  std::mutex host_mu;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t host_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // computed[2], copied[2]
  char* host_scratch = nullptr;
  size_t host_scratch_bytes = 0;
  unsigned next_counter = 0;
  int num_sms = 0;
  // polyphase small calls (cluster items): L2 exchange scratch, a ring of grow-only slots (a slot grows only in an
  // eager call: the first call of a size); tensor-core trajectory filter: K-split partial sums, two slots.  A slot
  // is reused after the launch that used it last (its event, SlotGuard); take and record happen under slot_mu.
  unsigned* poly_slab[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t poly_slab_words[4] = {0, 0, 0, 0};
  unsigned next_slab = 0;
  float* traj_part[2] = {nullptr, nullptr};
  size_t traj_part_words[2] = {0, 0};
  unsigned next_traj = 0;
  std::mutex slot_mu;
  cudaEvent_t slab_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t traj_ev[2] = {nullptr, nullptr};
  // gpurir_simulate_rir_batch: a ring of two grow-only pinned staging buffers for the job table, so the upload
  // is an asynchronous copy and the call returns without synchronising (a slot is reused once the copy that
  // last read it has executed: its event)
  std::mutex stage_mu;
  char* stage_host[2] = {nullptr, nullptr};
  size_t stage_bytes[2] = {0, 0};
  cudaEvent_t stage_done[2] = {nullptr, nullptr};
  unsigned stage_next = 0;
};
std::mutex g_mu;
constexpr int kMaxDevices = 64;
DeviceState g_dev[kMaxDevices];  // stable addresses: callers keep pointers while other threads add devices

DeviceState* device_state(int* err) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) { *err = cuda_fail(e, "cudaGetDevice"); return nullptr; }
  if (dev < 0 || dev >= kMaxDevices) { *err = GPURIR_EINVAL; return nullptr; }
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceState& d = g_dev[dev];
  if (!d.status) {
    e = cudaMalloc(&d.status, sizeof(int));
    if (e != cudaSuccess) { *err = cuda_fail(e, "cudaMalloc(status)"); return nullptr; }
    e = cudaMemset(d.status, 0, sizeof(int));
    if (e != cudaSuccess) { *err = cuda_fail(e, "cudaMemset(status)"); return nullptr; }
    e = cudaMalloc(&d.work_counter, kCounterRing * sizeof(int));
    if (e != cudaSuccess) { *err = cuda_fail(e, "cudaMalloc(counter)"); return nullptr; }
    e = cudaDeviceGetAttribute(&d.num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) { *err = cuda_fail(e, "num_sms"); return nullptr; }
  }
  *err = GPURIR_OK;
  return &d;
}

// Eq. 9 with the window argument 2 pi n / (Q fs T_w) (erratum C11).
double lut_entry(long long n, double Tw, double fs, int Q, long long half) {
  if (n < -half || n > half) return 0.0;
  double t = (double)n / (Q * fs);
  if (!(t > -Tw / 2 && t < Tw / 2)) return 0.0;  // open support (C8)
  double win = 0.5 * (1.0 + cos(2.0 * M_PI * (double)n / (Q * fs * Tw)));
  double arg = M_PI * (double)n / Q;
  return win * (n == 0 ? 1.0 : sin(arg) / arg);
}

long long lut_half(double Tw, double fs, int Q) { return (long long)ceil(Tw * Q * fs / 2.0 - 1e-9); }

// Phase-major interpolation table for the LUT kernel:
// TP[ph][jj + joff] = (T[Q jj + ph + 1], T[Q jj + ph] - T[Q jj + ph + 1]).
const LutEntry* ensure_lut(DeviceState* d, double Tw, double fs, int Q, double H, cudaStream_t stream, int* err) {
  *err = GPURIR_OK;
  for (const LutEntry& L : d->luts)
    if (L.Tw == Tw && L.fs == fs && L.Q == Q) return &L;
  long long half = lut_half(Tw, fs, Q);
  LutEntry L;
  L.Tw = Tw; L.fs = fs; L.Q = Q;
  L.joff = (int)ceil(H) + kS + 2;
  L.cols = 2 * L.joff + 1;
  L.rows = Q;
  std::vector<float2> tab((size_t)L.rows * L.cols);
  for (int ph = 0; ph < L.rows; ph++)
    for (int c = 0; c < L.cols; c++) {
      long long jj = c - L.joff;
      long long n = (long long)Q * jj + ph;
      double t0 = lut_entry(n, Tw, fs, Q, half), t1 = lut_entry(n + 1, Tw, fs, Q, half);
      tab[(size_t)ph * L.cols + c] = make_float2((float)t1, (float)(t0 - t1));
    }
  size_t bytes = tab.size() * sizeof(float2);
  cudaError_t e = cudaMalloc(&L.dev, bytes);
  if (e != cudaSuccess) { *err = cuda_fail(e, "cudaMalloc(lut)"); return nullptr; }
  e = cudaMemcpyAsync(L.dev, tab.data(), bytes, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // host staging vector goes out of scope
  if (e != cudaSuccess) { cudaFree(L.dev); *err = cuda_fail(e, "upload(lut)"); return nullptr; }
  d->luts.push_back(L);
  return &d->luts.back();
}

// Texture-LUT mode ("texture memory ... hardware interpolation"): T[n], n = -half..half,
// in a 1-D CUDA array, linear filtering, unnormalised coordinates, border addressing (0 outside the table).
const TexEntry* ensure_tex(DeviceState* d, double Tw, double fs, int Q, cudaStream_t stream, int* err) {
  *err = GPURIR_OK;
  for (const TexEntry& T : d->texs)
    if (T.Tw == Tw && T.fs == fs && T.Q == Q) return &T;
  TexEntry T;
  T.Tw = Tw; T.fs = fs; T.Q = Q;
  T.half = lut_half(Tw, fs, Q);
  const long long n = 2 * T.half + 1;
  int dev = 0, maxw = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxTexture1DWidth, dev);
  if (n > maxw) { *err = GPURIR_EINVAL; return nullptr; }
  std::vector<float> tab((size_t)n);
  for (long long i = -T.half; i <= T.half; i++) tab[(size_t)(i + T.half)] = (float)lut_entry(i, Tw, fs, Q, T.half);
  cudaChannelFormatDesc cd = cudaCreateChannelDesc<float>();
  cudaError_t e = cudaMallocArray(&T.arr, &cd, (size_t)n, 0);
  if (e != cudaSuccess) { *err = cuda_fail(e, "cudaMallocArray(lut tex)"); return nullptr; }
  e = cudaMemcpy2DToArrayAsync(T.arr, 0, 0, tab.data(), n * sizeof(float), n * sizeof(float), 1,
                               cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // the staging vector goes out of scope
  if (e != cudaSuccess) { cudaFreeArray(T.arr); *err = cuda_fail(e, "upload(lut tex)"); return nullptr; }
  cudaResourceDesc rd;
  memset(&rd, 0, sizeof(rd));
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = T.arr;
  cudaTextureDesc td;
  memset(&td, 0, sizeof(td));
  td.addressMode[0] = cudaAddressModeBorder;
  td.filterMode = cudaFilterModeLinear;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  e = cudaCreateTextureObject(&T.tex, &rd, &td, nullptr);
  if (e != cudaSuccess) { cudaFreeArray(T.arr); *err = cuda_fail(e, "cudaCreateTextureObject"); return nullptr; }
  d->texs.push_back(T);
  return &d->texs.back();
}

// Polyphase expansion of Eq. 6 (reading R11): for every integer tap m = k - floor(x) that the open support
// |k - x| < H can reach (m_lo = floor(-H) + 1 .. m_hi), delta'(m - phi) ~= sum_{d<8} P[m][d] T_d(2 phi - 1),
// phi in [0, 1), by the truncated Chebyshev series of the 64-node interpolant (max error 4.3e-7 for 16-96 kHz,
// integer or fractional H).  Rows are the kernel's taps mi = m - m_lo.
const int kPolyDeg = 8, kPolyNodes = 64, kPolyMaxTaps = 512;
double eq6_samples(double u, double H) {
  if (!(u > -H && u < H)) return 0.0;  // open support (C8)
  const double w = 0.5 * (1.0 + cos(M_PI * u / H));
  return w * (u == 0.0 ? 1.0 : sin(M_PI * u) / (M_PI * u));
}
// Host fit of R11: taps m_lo .. m_lo + ntaps - 1 (ntaps padded to a multiple of 8 with zero taps), table in
// the kernel's layout [channel pair q][tap mi][2].  Returns the padded tap count, or -EINVAL.
int poly_fit(double Tw, double fs, int* mlo_out, std::vector<float>& tab) {
  const double H = Tw * fs / 2.0;
  const int mlo = (int)floor(-H) + 1;
  const int mhi = (H == floor(H)) ? (int)H : (int)floor(H) + 1;
  const int ntaps = mhi - mlo + 1;
  const int npad = (ntaps + 7) & ~7;  // zero taps appended: the kernel's FIR runs in groups of 8 taps
  if (!(H > 0) || ntaps < 1 || npad > kPolyMaxTaps) return -GPURIR_EINVAL;
  tab.assign((size_t)npad * kPolyDeg, 0.f);
  for (int mi = 0; mi < ntaps; mi++) {
    const int m = mlo + mi;
    double c[kPolyDeg] = {0};
    for (int i = 0; i < kPolyNodes; i++) {
      const double th = M_PI * (i + 0.5) / kPolyNodes, y = cos(th), phi = 0.5 * (y + 1.0);
      const double fv = eq6_samples((double)m - phi, H);
      for (int k = 0; k < kPolyDeg; k++) c[k] += fv * cos(k * th);  // T_k(y) = cos(k theta)
    }
    // layout [channel pair q][tap mi][2]: the kernel's FIR group for pair q streams its taps contiguously
    for (int k = 0; k < kPolyChannels; k++)  // channels past kPolyChannels stay 0 (a shorter expansion)
      tab[((size_t)(k >> 1) * npad + mi) * 2 + (k & 1)] = (float)(c[k] * (k ? 2.0 : 1.0) / kPolyNodes);
  }
  *mlo_out = mlo;
  return npad;
}

// Eigen-decomposition of a symmetric 4 x 4 matrix by cyclic Jacobi rotations (fp64, to convergence): a = V
// diag(w) V^T, eigenvector k in column k of v.
static void jacobi4(double a[4][4], double w[4], double v[4][4]) {
  for (int i = 0; i < 4; i++)
    for (int j = 0; j < 4; j++) v[i][j] = i == j;
  for (int sweep = 0; sweep < 64; sweep++) {
    double off = 0.0;
    for (int p = 0; p < 4; p++)
      for (int q = p + 1; q < 4; q++) off += a[p][q] * a[p][q];
    if (off == 0.0) break;
    for (int p = 0; p < 4; p++)
      for (int q = p + 1; q < 4; q++) {
        if (a[p][q] == 0.0) continue;
        const double th = 0.5 * atan2(2.0 * a[p][q], a[q][q] - a[p][p]), c = cos(th), s = sin(th);
        for (int k = 0; k < 4; k++) {  // a <- a J (columns p, q), then J^T a (rows p, q)
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 4; k++) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 4; k++) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 4; i++) w[i] = a[i][i];
}

// Low-rank FIR of R11 (reading R13): the 8 channel filters P_d[m] restricted to the taps away from
// the centre have numerical rank 4 (the windowed sinc there is sin(pi phi) times a function of phi that varies
// slowly with m), so after an orthogonal change of channel basis G' = Q G — per parity (P_d[1 - m] =
// (-1)^d P_d[m], Eq. 6 is even, so Q is block diagonal over even / odd d), rows the eigenvectors of the far taps'
// Gram matrix sum_m P[m] P[m]^T by decreasing eigenvalue — only the rotated channels 0..3 need the whole support;
// channels 4..7 keep a window of nn = 8 taps, m = -3 .. 4, around m = 0, 1 (the coefficients dropped outside it
// are < 5e-8 of the peak at 8-96 kHz and T_w = 2-8 ms, against the expansion's 4.3e-7).  The kernel converts G, rotates it by Q and runs the FIR on
// 4 ntaps + 4 nn taps per output instead of 8 ntaps.  Device table: far [2 pairs][ntaps][2] (rotated channels
// (0, 1), (2, 3)), near [2 pairs][nn][2] (channels (4, 5), (6, 7)) for taps mi = nmi0 .. nmi0 + nn - 1, then
// Q [parity][k][i] (32 floats): rotated channel 2 k + par = sum_i Q[par][k][i] G_{2 i + par}, the k-th
// eigenvector of that parity.
void poly_fir_tables(const std::vector<float>& tab, int npad, int mlo, std::vector<float>& out, int* nmi0_out,
                     int* nn_out) {
  auto Pd = [&](int mi, int d) { return (double)tab[((size_t)(d >> 1) * npad + mi) * 2 + (d & 1)]; };
  const int mc = -mlo;                         // tap index of m = 0
  // the window: m = -3 .. 4 for tables of <= 64 taps (the kernel's fixed-stride variant: unaligned near refills);
  // longer tables keep an aligned window of 16 (or 24) taps covering m = -6 .. 7, split over the FIR's tap halves
  // (measured: the unaligned 8-tap window cost config 4 at 48 kHz 14 % while saving 1.9 % at 16 kHz)
  int nmi0, nn;
  if (npad <= 64) {
    nn = std::min(8, npad);
    nmi0 = std::max(0, std::min(mc - 3, npad - nn));
  } else {
    nmi0 = std::max(0, ((mc - 6) / 8) * 8);
    nn = std::min(npad - nmi0, ((mc + 8 - nmi0 + 7) / 8) * 8);
  }
  double Q[8][8] = {};
  for (int par = 0; par < 2; par++) {
    double a[4][4] = {}, w[4], v[4][4];
    for (int mi = 0; mi < npad; mi++) {
      if (mi >= nmi0 && mi < nmi0 + nn) continue;
      for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) a[i][j] += Pd(mi, 2 * i + par) * Pd(mi, 2 * j + par);
    }
    jacobi4(a, w, v);
    int ord[4] = {0, 1, 2, 3};
    std::sort(ord, ord + 4, [&](int x, int y) { return w[x] > w[y]; });
    for (int k = 0; k < 4; k++)
      for (int i = 0; i < 4; i++) Q[2 * k + par][2 * i + par] = v[i][ord[k]];
  }
  auto Pr = [&](int mi, int r) {  // rotated coefficient P'_r[mi] = sum_d Q[r][d] P_d[mi]
    double s = 0.0;
    for (int d = 0; d < 8; d++) s += Q[r][d] * Pd(mi, d);
    return (float)s;
  };
  out.assign((size_t)4 * npad + (size_t)4 * nn + 32, 0.f);
  for (int q = 0; q < 2; q++)
    for (int mi = 0; mi < npad; mi++)
      for (int c = 0; c < 2; c++) out[((size_t)q * npad + mi) * 2 + c] = Pr(mi, 2 * q + c);
  float* near = out.data() + (size_t)4 * npad;
  for (int q = 0; q < 2; q++)
    for (int i = 0; i < nn; i++)
      for (int c = 0; c < 2; c++) near[((size_t)q * nn + i) * 2 + c] = Pr(nmi0 + i, 4 + 2 * q + c);
  float* Qo = near + (size_t)4 * nn;  // [parity][k][i]: rotated channel 2 k + par = sum_i Q G_{2 i + par}
  for (int par = 0; par < 2; par++)
    for (int k = 0; k < 4; k++)
      for (int i = 0; i < 4; i++) Qo[(par * 4 + k) * 4 + i] = (float)Q[2 * k + par][2 * i + par];
  *nmi0_out = nmi0;
  *nn_out = nn;
}

const PolyEntry* ensure_poly(DeviceState* d, double Tw, double fs, cudaStream_t stream, int* err) {
  *err = GPURIR_OK;
  for (const PolyEntry& P : d->polys)
    if (P.Tw == Tw && P.fs == fs) return &P;
  PolyEntry P;
  P.Tw = Tw; P.fs = fs;
  std::vector<float> tab0, tab;
  P.ntaps = poly_fit(Tw, fs, &P.mlo, tab0);
  if (P.ntaps < 0) { *err = GPURIR_EINVAL; return nullptr; }
  poly_fir_tables(tab0, P.ntaps, P.mlo, tab, &P.nmi0, &P.nn);
  const size_t bytes = tab.size() * sizeof(float);
  cudaError_t e = cudaMalloc(&P.dev, bytes);
  if (e != cudaSuccess) { *err = cuda_fail(e, "cudaMalloc(poly)"); return nullptr; }
  e = cudaMemcpyAsync(P.dev, tab.data(), bytes, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);  // the staging vector goes out of scope
  if (e != cudaSuccess) { cudaFree(P.dev); *err = cuda_fail(e, "upload(poly)"); return nullptr; }
  d->polys.push_back(P);
  return &d->polys.back();
}

// Polyphase fixed-point width (ism_poly_kernel.cu, poly_add): a shoebox lattice holds one image per room
// volume V, so about 4 pi d^2 (c / fs) / V images share one integer sample position at distance d.  With twice
// that at the farthest ISM delay (+16) as the bound N, single-word accumulation with bits = 22 is used when
// 2^22 N <= 2^30 (N <= 256); otherwise 0 selects the two-word scheme (2^28 resolution).
#ifndef GPURIR_FUSE_MIN_PER_SM
#define GPURIR_FUSE_MIN_PER_SM 0  // RIRs per SM from which the polyphase kernel writes the diffuse tail itself
                                  // (A/B: fusing is faster at every M from 12 to 2048, so always)
#endif
constexpr long long kHostChunkMin = 2048;  // RIRs per chunk of gpurir_simulate_rir_host (fills the GPU)

// Polyphase fixed point (ism_poly_kernel.cu, tile setup): a tile needs the two-word scheme when its bound on
// the images per sample position, N = 8 pi x_hi^2 / V_s + 24 x_hi / L_min + 16 (x_hi the tile's largest delay,
// V_s the room volume and L_min its shortest side, all in samples), reaches 2^12.  The call allocates the
// fine plane when its last tile could.
bool poly_two_word_for(const float L[3], long long nISM, double fs, double c, double Tw) {
  const double k = fs / c;
  const double Vs = (double)L[0] * L[1] * L[2] * k * k * k;
  const double Lmin = std::min(std::min((double)L[0], (double)L[1]), (double)L[2]) * k;
  const double xhi = (double)nISM + Tw * fs / 2.0 + 1.0;
  return 8.0 * M_PI * xhi * xhi / Vs + 24.0 * xhi / Lmin + 16.0 >= 4096.0;  // the kernel's lb >= 13: bits < 18
}

// Mode tables of one call (LUT: phase-major smem table; texture LUT: filtered texture; polyphase table).
int setup_mode(DeviceState* d, const gpurir_opts& o, double fs, double H, cudaStream_t stream, IsmArgs& A) {
  int st = GPURIR_OK;
  std::lock_guard<std::mutex> lk(g_mu);
  if (o.mode == GPURIR_LUT) {
    const LutEntry* L = ensure_lut(d, o.Tw, fs, o.lut_Q, H, stream, &st);
    if (!L) return st;
    A.lut = L->dev; A.lut_rows = L->rows; A.lut_cols = L->cols; A.lut_joff = L->joff;
    A.lutQ = o.lut_Q;
  } else if (o.mode == GPURIR_LUT_TEX) {
    const TexEntry* T = ensure_tex(d, o.Tw, fs, o.lut_Q, stream, &st);
    if (!T) return st;
    A.tex = (unsigned long long)T->tex;
    A.texQ = (float)o.lut_Q;
    A.tex_off = (float)((double)T->half + 0.5);
  } else if (o.mode == GPURIR_POLY) {
    const PolyEntry* P = ensure_poly(d, o.Tw, fs, stream, &st);
    if (!P) return st;
    A.poly_P = P->dev; A.poly_ntaps = P->ntaps; A.poly_mlo = P->mlo; A.poly_nmi0 = P->nmi0; A.poly_nn = P->nn;
    A.poly_i2d_bias = 4503601774854144.0;
    A.poly_m1 = -1.f;
  }
  return GPURIR_OK;
}

int validate_mode(const gpurir_opts& o) {
  if (o.mode < GPURIR_FP32 || o.mode > GPURIR_POLY) return GPURIR_EINVAL;
  if (o.mode == GPURIR_LUT && (o.lut_Q & (o.lut_Q - 1))) return GPURIR_EINVAL;  // power of two (R4)
  return GPURIR_OK;
}

double sabine(const float L[3], const float b[6]) {
  double V = (double)L[0] * L[1] * L[2];
  double S[6] = {(double)L[1] * L[2], (double)L[1] * L[2], (double)L[0] * L[2],
                 (double)L[0] * L[2], (double)L[0] * L[1], (double)L[0] * L[1]};
  double den = 0.0;
  for (int i = 0; i < 6; i++) den += S[i] * (1.0 - (double)b[i] * b[i]);
  if (den <= 0.0) return INFINITY;
  return 0.161 * V / den;
}

// log2 |beta_w| and sign / zero masks of the six walls, shared by every image of a room.
void beta_logs(const float b[6], float lb[6], unsigned* neg, unsigned* zero) {
  *neg = 0; *zero = 0;
  for (int w = 0; w < 6; w++) {
    if (b[w] < 0.f) *neg |= 1u << w;
    if (b[w] == 0.f) { *zero |= 1u << w; lb[w] = 0.f; }
    else lb[w] = (float)log2(fabs((double)b[w]));
  }
}

int validate_room(const float L[3], const float b[6], const int nb[3], int pattern) {
  for (int i = 0; i < 3; i++) {
    if (!(L[i] > 0.f) || !isfinite(L[i])) return GPURIR_EINVAL;
    if (nb[i] < 1) return GPURIR_EINVAL;
  }
  for (int i = 0; i < 6; i++)
    if (!(fabsf(b[i]) <= 1.f)) return GPURIR_EINVAL;
  if (pattern < 0 || pattern > 4) return GPURIR_EINVAL;
  return GPURIR_OK;
}

// Reciprocals the polyphase tile setup multiplies by (device divisions are long fp64 sequences on one thread):
// 1/L[0..2] (m^-1), 1/V_s with V_s the room volume in samples^3, 1/L_min,s (the shortest side in samples)
void poly_geo_consts(const float L[3], double fs_over_c, double geo[5]) {
  for (int i = 0; i < 3; i++) geo[i] = 1.0 / (double)L[i];
  const double Vs = (double)L[0] * (double)L[1] * (double)L[2] * fs_over_c * fs_over_c * fs_over_c;
  const double Lmin_s = fmin(fmin((double)L[0], (double)L[1]), (double)L[2]) * fs_over_c;
  geo[3] = 1.0 / Vs;
  geo[4] = 1.0 / Lmin_s;
}

void fill_common(IsmArgs& A, double fs, double c, double Tw) {
  A.fs_over_c = fs / c;
  A.c_over_fs = c / fs;
  double H = Tw * fs / 2.0;
  A.H = (float)H;
  A.invH = (float)(1.0 / H);
  A.nbw = (int)floor(((double)kS - 1.0 + 2.0 * H) / kS) + 1;
  double Hs = exp2(ceil(log2(H)));
  double rho = H / Hs, r2 = rho * rho;
  A.invHs = (float)(1.0 / Hs);
  A.rho2 = (float)r2;
  const double b[3] = {kWb0, kWb1, kWb2};
  for (int i = 0; i < 3; i++) A.wb[i] = (float)(b[i] / pow(r2, i + 1));
  // c(sigma) = sigma (wb0 + wb1 sigma + wb2 sigma^2) rewritten in u = 1 + sigma, which the kernel clamps to
  // [0, 1] with FFMA.SAT (u = 1 <=> the window edge): a_j = sum_k wb_{k-1} C(k,j) (-1)^(k-j)
  double a[4] = {0, 0, 0, 0};
  for (int k = 1; k <= 3; k++) {
    double ck = 1.0;  // C(k, j)
    for (int j = 0; j <= k; j++) {
      a[j] += (double)A.wb[k - 1] * ck * (((k - j) & 1) ? -1.0 : 1.0);
      ck = ck * (double)(k - j) / (double)(j + 1);
    }
  }
  for (int j = 1; j <= 3; j++) A.wa[j] = (float)a[j];
  float s = A.wa[3];  // Horner at u = 1 in fp32, so that c(1) = 0 exactly on the device
  s = s + A.wa[2];
  s = s + A.wa[1];
  A.wa[0] = -s;
  A.urho = (float)(1.0 - r2);
  // Eq. 11 coefficients, argument rescaled from u/(2H) to u/(2Hs)
  A.hc[0] = (float)(-4.93359375 / r2);
  A.hc[1] = (float)(4.04296875 / (r2 * r2));
  A.hc[2] = (float)(-1.2294921875 / (r2 * r2 * r2));
  A.x2clamp = (float)(r2 / 4.0);
}

int auto_split(long long nclusters, int requested) {
  if (requested > 0) return requested > kMaxSplit ? kMaxSplit : requested;
  int s = 1;
  while (s < kMaxSplit && nclusters * s < 148LL * 4) s *= 2;
  return s;
}

// Stream order for a scratch slot shared round-robin by calls on any stream: the call that takes the slot waits
// (on its stream) for the event its previous user recorded after its launch, and records the slot's event after its
// own launch (SlotGuard's destructor); the device's slot_mu is held from take to record, so no two calls interleave.
// A stream being captured into a CUDA graph neither waits nor records (a graph replays its nodes in order).
struct SlotGuard {
  std::unique_lock<std::mutex> lk;
  cudaEvent_t* ev = nullptr;  // the slot's event (created on first use)
  cudaStream_t stream = nullptr;
  bool capturing = false;
  void take(std::mutex& mu, cudaEvent_t* slot_ev, cudaStream_t s) {
    lk = std::unique_lock<std::mutex>(mu);
    ev = slot_ev;
    stream = s;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    capturing = cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone;
    if (!capturing && *ev) cudaStreamWaitEvent(s, *ev, 0);
  }
  ~SlotGuard() {
    if (!ev || capturing) return;
    if (!*ev && cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess) { *ev = nullptr; return; }
    cudaEventRecord(*ev, stream);
  }
};

// Grows every slot of a round-robin scratch ring to at least `need` elements (with headroom for the next call
// size) when the one about to be taken is short, so that after one eager call of a size every later call of that
// size — whichever slot it draws, on whichever stream, captured or not — allocates nothing.  Slots may still be in
// use by earlier launches on other streams: the device is synchronised before any is freed.  A stream being
// captured cannot allocate or synchronise: the call fails with GPURIR_ECUDA and a message instead of invalidating
// the capture (gpurir.h: capture after one eager call of the same size).
template <class T>
int grow_ring(T** slot, size_t* words, int n, size_t need, bool capturing, const char* what) {
  bool short_any = false, held = false;
  for (int i = 0; i < n; i++) { short_any |= words[i] < need; held |= slot[i] != nullptr; }
  if (!short_any) return GPURIR_OK;
  if (capturing) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: scratch must grow during stream capture; make one eager call "
             "of this size first", what);
    return GPURIR_ECUDA;
  }
  if (held) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, what);
  }
  const size_t w = need + need / 4;
  for (int i = 0; i < n; i++) {
    if (words[i] >= need) continue;
    if (slot[i]) {
      cudaError_t e = cudaFree(slot[i]);
      if (e != cudaSuccess) return cuda_fail(e, what);
      slot[i] = nullptr;
      words[i] = 0;
    }
    cudaError_t e = cudaMalloc((void**)&slot[i], w * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, what);
    words[i] = w;
  }
  return GPURIR_OK;
}

// Exchange scratch of a cluster-item polyphase launch (ism_poly_kernel.cu: the ranks' planes meet through L2).
// Fully overwritten by each launch, so never zeroed.
int set_poly_slab(DeviceState* d, IsmArgs& A, long long n_work, int split, cudaStream_t stream, SlotGuard& guard) {
  const int S = ism_poly_cluster_size(n_work, d->num_sms, split, A.poly_ntaps, A.poly_gbz != 0, nullptr);
  if (S <= 0) return GPURIR_OK;
  const size_t need = ism_poly_slab_words(n_work, S, A.poly_ntaps, d->num_sms);
  unsigned k;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    k = d->next_slab++ % 4;
  }
  guard.take(d->slot_mu, &d->slab_ev[k], stream);
  if (int st = grow_ring(d->poly_slab, d->poly_slab_words, 4, need, guard.capturing, "poly slab")) return st;
  A.poly_slab = d->poly_slab[k];
  A.poly_slab_w = (kPolyTile + A.poly_ntaps - 1 + 31) & ~31;
  return GPURIR_OK;
}

// Work-queue head for one persistent launch: a ring of kCounterRing counters so that up to that many
// calls can be in flight on different streams (each is zeroed on its stream right before its launch).
int* take_counter(DeviceState* d) {
  std::lock_guard<std::mutex> lk(g_mu);
  return d->work_counter + (d->next_counter++ % kCounterRing);
}

// Persistent warp-specialised kernel when there are enough (RIR, tile) work items to keep one CTA per
// SM busy; the cluster-split kernel otherwise (latency-bound small calls).  split < 0 forces persistent.
bool use_persistent(long long n_work, int split, int num_sms) {
  if (split < 0) return true;
  if (split > 0) return false;
  return n_work >= 4LL * num_sms;
}

// The polyphase kernel writes the diffuse tail of the RIRs it finishes; GPURIR_FUSE_TAIL=0 in the
// environment keeps tail_kernel instead (A/B measurements only)
bool fuse_tail_enabled() {
  static const int v = [] {
    const char* e = getenv("GPURIR_FUSE_TAIL");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  return v != 0;
}

int status_code(int s) {
  if (s & kStatusDegenerate) return GPURIR_EDEGENERATE;
  if (s & kStatusCapacity) return GPURIR_ECAPACITY;
  return GPURIR_EINVAL;
}

int* status_ptr(const gpurir_opts& o, DeviceState* d) { return o.status ? o.status : d->status; }

int finish(const gpurir_opts& o, cudaStream_t st, DeviceState* d) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "launch");
  if (o.flags & GPURIR_FLAG_SYNC) {
    int* sp = status_ptr(o, d);
    int s = 0;
    e = cudaMemcpyAsync(&s, sp, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "sync");
    if (s) {
      cudaMemsetAsync(sp, 0, sizeof(int), st);
      return status_code(s);
    }
  }
  return GPURIR_OK;
}

// GPURIR_PLAN_TIMING=1: the batch call prints its host phases (plan, workspace, staging, launch) to stderr
bool plan_timing() {
  static const bool on = [] {
    const char* e = getenv("GPURIR_PLAN_TIMING");
    return e && atoi(e) != 0;
  }();
  return on;
}
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Host plan of a multi-room batch (gpurir_simulate_rir_batch, gpurir_workspace_bytes): the device job table, the
// heavy-first tile list of the ISM kernel and the chunk list of the tail kernel.
struct BatchPlan {
  std::vector<BatchJob> jobs;
  std::vector<int2> tiles, chunks;
  bool poly = false, persistent = false, any_two_word = false, fused = false;
  int kmode = 0;
  size_t off_tiles = 0, off_chunks = 0, bytes = 0;  // device workspace layout
  std::vector<int> ntile;                            // scratch: tiles per room
  // a plan is reused by the next call on the same host thread (thread_local in the callers): its vectors keep
  // their capacity, so a large batch does not map and zero-fill ~24 MB of fresh pages on every call
  void reset() {
    tiles.clear(); chunks.clear();
    poly = persistent = any_two_word = fused = false;
    kmode = 0;
    off_tiles = off_chunks = bytes = 0;
  }
};

int plan_batch(int n_rooms, const gpurir_room* rooms, double fs, double c, const gpurir_opts& o, int num_sms,
               BatchPlan& P) {
  if (n_rooms <= 0 || !rooms || !(fs > 0) || !(c > 0)) return GPURIR_EINVAL;
  if (int em = validate_mode(o)) return em;
  const double H = o.Tw * fs / 2.0;
  if ((int)ceil((kTCPersistent + 2.0 * H) / kS) + 1 > kMaxBins) return GPURIR_EINVAL;
  P.jobs.resize(n_rooms);
  // rooms [lo, hi): validation and the job record of each (independent per room); the first invalid room's code
  struct Part {
    int err = GPURIR_OK, err_room = 0;
    bool two_word = false;
    long long small_tiles = 0;  // work items at the cluster kernel's tile length (kernel choice)
  };
  auto plan_rooms = [&](int lo, int hi, Part& out) {
    for (int i = lo; i < hi; i++) {
      const gpurir_room& R = rooms[i];
      int e0 = validate_room(R.room_sz, R.beta, R.nb_img, R.mic_pattern);
      if (!e0 && (R.spkr_pattern < 0 || R.spkr_pattern > 4)) e0 = GPURIR_EINVAL;
      if (!e0 && (!(R.Tmax > 0) || !(R.Tdiff >= 0) || R.out_offset < 0)) e0 = GPURIR_EINVAL;
      long long nS = 0, nISM = 0;
      if (!e0) {
        nS = gpurir_nsamples(R.Tmax, fs);
        nISM = std::min(gpurir_nsamples(R.Tdiff, fs), nS);
        if (nS > (1LL << 30) || nISM > kMaxIsmSamples) e0 = GPURIR_EINVAL;
      }
      if (e0) { out.err = e0; out.err_room = i; return; }
      BatchJob& J = P.jobs[i];
      memset(&J, 0, sizeof(J));
      for (int a = 0; a < 3; a++) {
        J.L[a] = R.room_sz[a]; J.src[a] = R.pos_src[a]; J.rcv[a] = R.pos_rcv[a]; J.orv[a] = R.orV_rcv[a];
        J.ors[a] = R.orV_src[a];
        J.nb[a] = R.nb_img[a];
      }
      for (int w = 0; w < 6; w++) J.beta[w] = R.beta[w];
      beta_logs(R.beta, J.lb, &J.neg, &J.zero);
      J.pattern = R.mic_pattern;
      J.spkr_pattern = R.spkr_pattern;
      J.nISM = (int)nISM; J.nS = (int)nS; J.out_offset = R.out_offset;
      const double T60 = sabine(R.room_sz, R.beta);
      J.kappa_fs = isinf(T60) ? 0.f : (float)(6.0 * log(10.0) / T60 / fs);  // Eq. 8, reading C14
      J.rir_global = o.rir_index_base + R.rir_index;                        // reading C16: global stream id
      poly_geo_consts(R.room_sz, fs / c, J.geo);
      out.two_word = out.two_word || poly_two_word_for(R.room_sz, nISM, fs, c, o.Tw);
      out.small_tiles += (nISM + kTC - 1) / kTC;
    }
  };
  // large batches (dataset generation, config 5) over host threads: the plan of 100 000 rooms is ~11 ms on one
  // core, which a slower or busier host turns into the step's bottleneck (the kernel takes ~25 ms); small calls
  // stay on the calling thread.  GPURIR_PLAN_THREADS caps the count (1 = serial).
  static const int max_threads = [] {
    const char* e = getenv("GPURIR_PLAN_THREADS");
    const int hw = (int)std::thread::hardware_concurrency();
    const int x = e ? atoi(e) : std::min(8, std::max(1, hw));
    return std::max(1, x);
  }();
  const int nt = std::max(1, std::min(max_threads, n_rooms / 4096));
  std::vector<Part> parts((size_t)nt);
  if (nt == 1) {
    plan_rooms(0, n_rooms, parts[0]);
  } else {
    std::vector<std::thread> th;
    th.reserve((size_t)nt - 1);
    const int per = (n_rooms + nt - 1) / nt;
    for (int t = 1; t < nt; t++)
      th.emplace_back(plan_rooms, t * per, std::min(n_rooms, (t + 1) * per), std::ref(parts[(size_t)t]));
    plan_rooms(0, std::min(n_rooms, per), parts[0]);
    for (auto& x : th) x.join();
  }
  long long small_tiles = 0;
  for (const Part& pt : parts)  // in room order: the first invalid room decides the code, as serially
    if (pt.err) return pt.err;
  for (const Part& pt : parts) {
    P.any_two_word = P.any_two_word || pt.two_word;
    small_tiles += pt.small_tiles;
  }
  P.poly = o.mode == GPURIR_POLY;
  P.kmode = o.mode == GPURIR_POLY ? (P.poly ? GPURIR_POLY : GPURIR_FP32) : o.mode;
  P.persistent = P.poly || use_persistent(small_tiles, o.split, num_sms);
  // polyphase: every room's diffuse tail is written by the CTA that finishes its last (end-aligned) ISM tile,
  // which holds the whole 10 ms envelope window (fs <= 102.4 kHz); rooms without ISM samples keep tail_kernel
  P.fused = P.poly && llround(0.010 * fs) <= kPolyTile && fuse_tail_enabled();
  for (int i = 0; i < n_rooms; i++) {
    const BatchJob& J = P.jobs[i];
    if (J.nISM >= J.nS || (P.fused && J.nISM > 0)) continue;
    const long long groups = (J.nS + 3) / 4 - J.nISM / 4;
    const int nch = (int)((groups + kTailChunk / 4 - 1) / (kTailChunk / 4));
    for (int ch = 0; ch < nch; ch++) P.chunks.push_back(make_int2(i, ch));
  }
  const int tile_len = P.poly ? kPolyTile : P.persistent ? kTCPersistent : kTC;
  std::vector<int>& ntile = P.ntile;
  ntile.resize(n_rooms);
  int max_tiles = 0;
  size_t total_tiles = 0;
  for (int i = 0; i < n_rooms; i++) {
    ntile[i] = (P.jobs[i].nISM + tile_len - 1) / tile_len;
    max_tiles = std::max(max_tiles, ntile[i]);
    total_tiles += (size_t)ntile[i];
  }
  P.tiles.reserve(total_tiles);
  // heavy-first without a comparison sort: image density grows ~ t^2 (SURVEY §7 hard part 2), so emit the tiles
  // by decreasing end sample (a counting order over tile-length buckets).  The polyphase kernel's tiles are
  // end-aligned per room (tile t of n ends at nISM - (n - 1 - t) 1024); the other kernels' start at t tile_len.
  if (P.poly) {
    std::vector<size_t> start(max_tiles + 1, 0);  // bucket = ceil(te / tile_len) - 1, emitted in decreasing order
    auto bucket = [&](int i, int t) {
      const int te = P.jobs[i].nISM - (ntile[i] - 1 - t) * tile_len;
      return max_tiles - 1 - ((te + tile_len - 1) / tile_len - 1);  // 0 = the latest end
    };
    for (int i = 0; i < n_rooms; i++)
      for (int t = 0; t < ntile[i]; t++) start[bucket(i, t) + 1]++;
    for (int b = 0; b < max_tiles; b++) start[b + 1] += start[b];
    P.tiles.resize(total_tiles);
    for (int i = 0; i < n_rooms; i++)
      for (int t = ntile[i] - 1; t >= 0; t--) P.tiles[start[bucket(i, t)]++] = make_int2(i, t);
  } else {
    for (int t = max_tiles - 1; t >= 0; t--)
      for (int i = 0; i < n_rooms; i++)
        if (ntile[i] > t) P.tiles.push_back(make_int2(i, t));
  }
  const size_t bj = P.jobs.size() * sizeof(BatchJob), bt = P.tiles.size() * sizeof(int2);
  P.off_tiles = (bj + 255) & ~(size_t)255;
  P.off_chunks = P.off_tiles + ((bt + 255) & ~(size_t)255);
  P.bytes = P.off_chunks + P.chunks.size() * sizeof(int2) + 256;
  return GPURIR_OK;
}

}  // namespace

extern "C" {

void gpurir_opts_default(gpurir_opts* o) {
  memset(o, 0, sizeof(*o));
  o->mode = GPURIR_FP32;
  o->Tw = 4e-3;
  o->lut_Q = 16;
}

long long gpurir_nsamples(double T, double fs) {
  long long n = (long long)ceil(T * fs - 1e-6);  // reading C9
  return n < 0 ? 0 : n;
}

double gpurir_sabine_t60(const float room_sz[3], const float beta[6]) { return sabine(room_sz, beta); }

int gpurir_beta_sabine(const float room_sz[3], double T60, int sign, int clamp, float beta_out[6], int* clamped) {
  if (clamped) *clamped = 0;
  if (!(T60 > 0.0)) return GPURIR_EINVAL;
  for (int i = 0; i < 3; i++)
    if (!(room_sz[i] > 0.f)) return GPURIR_EINVAL;
  double Lx = room_sz[0], Ly = room_sz[1], Lz = room_sz[2];
  double V = Lx * Ly * Lz, S = 2.0 * (Lx * Ly + Lx * Lz + Ly * Lz);
  double alpha = 0.161 * V / (T60 * S);
  if (alpha > 1.0) {
    if (!clamp) return GPURIR_EINFEASIBLE;
    if (clamped) *clamped = 1;
    for (int i = 0; i < 6; i++) beta_out[i] = 0.f;
    return GPURIR_OK;
  }
  float b = (float)(sqrt(1.0 - alpha) * (sign < 0 ? -1.0 : 1.0));
  for (int i = 0; i < 6; i++) beta_out[i] = b;
  return GPURIR_OK;
}

int gpurir_beta_sabine_weighted(const float room_sz[3], double T60, const float weights[6], int sign, int clamp,
                                float beta_out[6], int* clamped) {
  if (clamped) *clamped = 0;
  if (!(T60 > 0.0) || !weights) return GPURIR_EINVAL;
  for (int i = 0; i < 3; i++)
    if (!(room_sz[i] > 0.f)) return GPURIR_EINVAL;
  double Lx = room_sz[0], Ly = room_sz[1], Lz = room_sz[2];
  const double S[6] = {Ly * Lz, Ly * Lz, Lx * Lz, Lx * Lz, Lx * Ly, Lx * Ly};
  double Sw = 0.0;
  for (int i = 0; i < 6; i++) {
    if (!(weights[i] >= 0.f)) return GPURIR_EINVAL;
    Sw += S[i] * (double)weights[i];
  }
  if (!(Sw > 0.0)) return GPURIR_EINVAL;
  const double alpha0 = 0.161 * Lx * Ly * Lz / (T60 * Sw);  // Eq. 7 met exactly (reading R9)
  double alpha[6];
  bool infeasible = false;
  for (int i = 0; i < 6; i++) {
    alpha[i] = (double)weights[i] * alpha0;
    if (alpha[i] > 1.0) infeasible = true;
  }
  if (infeasible) {
    if (!clamp) return GPURIR_EINFEASIBLE;
    if (clamped) *clamped = 1;
    for (int i = 0; i < 6; i++) beta_out[i] = 0.f;
    return GPURIR_OK;
  }
  for (int i = 0; i < 6; i++) beta_out[i] = (float)(sqrt(1.0 - alpha[i]) * (sign < 0 ? -1.0 : 1.0));
  return GPURIR_OK;
}

double gpurir_att2t_sabine(double att_dB, double T60) { return att_dB / 60.0 * T60; }

int gpurir_t2n(double T, const float room_sz[3], double c, int nb_img_out[3]) {
  if (!(T > 0.0) || !(c > 0.0)) return GPURIR_EINVAL;
  for (int i = 0; i < 3; i++) {
    if (!(room_sz[i] > 0.f)) return GPURIR_EINVAL;
    nb_img_out[i] = 2 * ((int)ceil(c * T / (double)room_sz[i]) + 1) + 1;
  }
  return GPURIR_OK;
}

int gpurir_poly_table(double Tw, double fs, int* mlo, float* P_out, long long cap) {
  std::vector<float> tab;
  int m0 = 0;
  const int ntaps = poly_fit(Tw, fs, &m0, tab);
  if (ntaps < 0) return ntaps;
  if (mlo) *mlo = m0;
  if (P_out) {
    if (cap < (long long)ntaps * kPolyDeg) return -GPURIR_EINVAL;
    for (int mi = 0; mi < ntaps; mi++)  // [tap][channel] for the caller
      for (int k = 0; k < kPolyDeg; k++) P_out[(size_t)mi * kPolyDeg + k] = tab[((size_t)(k >> 1) * ntaps + mi) * 2 + (k & 1)];
  }
  return ntaps;
}

int gpurir_poly_fir_table(double Tw, double fs, int* mlo, int* nmi0, int* nn, float* out, long long cap) {
  std::vector<float> tab0, tab;
  int m0 = 0, a = 0, b = 0;
  const int ntaps = poly_fit(Tw, fs, &m0, tab0);
  if (ntaps < 0) return ntaps;
  poly_fir_tables(tab0, ntaps, m0, tab, &a, &b);
  if (mlo) *mlo = m0;
  if (nmi0) *nmi0 = a;
  if (nn) *nn = b;
  if (out) {
    if (cap < (long long)tab.size()) return -GPURIR_EINVAL;
    memcpy(out, tab.data(), tab.size() * sizeof(float));
  }
  return ntaps;
}

long long gpurir_lut_table(double Tw, double fs, int Q, float* lut_out, long long cap) {
  if (!(Tw > 0) || !(fs > 0) || Q < 1) return -GPURIR_EINVAL;
  long long half = lut_half(Tw, fs, Q);
  if (lut_out) {
    if (cap < 2 * half + 1) return -GPURIR_EINVAL;
    for (long long n = -half; n <= half; n++) lut_out[n + half] = (float)lut_entry(n, Tw, fs, Q, half);
  }
  return half;
}

int gpurir_simulate_rir(const float room_sz[3], const float beta[6], const float* pos_src, int M_src,
                        const float* pos_rcv, int M_rcv, const float* orV_rcv, int mic_pattern, const int nb_img[3],
                        double Tdiff, double Tmax, double fs, double c, float* out, const gpurir_opts* opts) {
  return gpurir_simulate_rir_dir(room_sz, beta, pos_src, M_src, nullptr, GPURIR_OMNI, pos_rcv, M_rcv, orV_rcv,
                                 mic_pattern, nb_img, Tdiff, Tmax, fs, c, out, opts);
}

int gpurir_simulate_rir_dir(const float room_sz[3], const float beta[6], const float* pos_src, int M_src,
                            const float* orV_src, int spkr_pattern, const float* pos_rcv, int M_rcv,
                            const float* orV_rcv, int mic_pattern, const int nb_img[3], double Tdiff, double Tmax,
                            double fs, double c, float* out, const gpurir_opts* opts) {
  gpurir_opts o;
  if (opts) o = *opts; else gpurir_opts_default(&o);
  if (!(o.Tw > 0)) o.Tw = 4e-3;
  if (o.lut_Q <= 0) o.lut_Q = 16;
  if (M_src <= 0 || M_rcv <= 0 || !pos_src || !pos_rcv || !out) return GPURIR_EINVAL;
  if (!(fs > 0) || !(c > 0) || !(Tmax > 0) || !(Tdiff >= 0)) return GPURIR_EINVAL;
  int st = validate_room(room_sz, beta, nb_img, mic_pattern);
  if (st) return st;
  if (mic_pattern != GPURIR_OMNI && !orV_rcv) return GPURIR_EINVAL;
  if (spkr_pattern < 0 || spkr_pattern > 4 || (spkr_pattern != GPURIR_OMNI && !orV_src)) return GPURIR_EINVAL;
  if (int em = validate_mode(o)) return em;
  double H = o.Tw * fs / 2.0;
  if ((int)ceil((kTCPersistent + 2.0 * H) / kS) + 1 > kMaxBins) return GPURIR_EINVAL;  // window too long
  long long nS = gpurir_nsamples(Tmax, fs);
  long long nISM = gpurir_nsamples(Tdiff, fs);
  if (nISM > nS) nISM = nS;
  if (nS > (1LL << 30) || nISM > kMaxIsmSamples) return GPURIR_EINVAL;
  long long M = (long long)M_src * M_rcv;
  if (M > (1LL << 30)) return GPURIR_EINVAL;

  DeviceState* d = device_state(&st);
  if (!d) return st;
  cudaStream_t stream = (cudaStream_t)o.stream;

  bool fused_tail = false;
  if (nISM > 0) {
    IsmArgs A;
    memset(&A, 0, sizeof(A));
    for (int i = 0; i < 3; i++) { A.L[i] = room_sz[i]; A.nb[i] = nb_img[i]; }
    for (int i = 0; i < 6; i++) A.beta[i] = beta[i];
    beta_logs(beta, A.lb, &A.neg, &A.zero);
    A.pattern = mic_pattern;
    A.pos_src = pos_src; A.pos_rcv = pos_rcv; A.orv = mic_pattern == GPURIR_OMNI ? nullptr : orV_rcv;
    A.ors = spkr_pattern == GPURIR_OMNI ? nullptr : orV_src;
    A.spkr_pattern = spkr_pattern;
    A.M_src = M_src; A.M_rcv = M_rcv; A.M = (int)M;
    A.invM = 1.0 / (double)M;
    A.invMrcv = 1.0 / (double)M_rcv;
    A.nISM = (int)nISM;
    A.row_stride = nS;
    poly_geo_consts(room_sz, fs / c, A.poly_geo);
    // polyphase mode runs the polyphase kernel at every call size: small calls split each tile's columns over a
    // thread-block cluster (ism_poly_kernel.cu), with the same bits as the persistent kernel
    const bool poly = o.mode == GPURIR_POLY;
    const int kmode = o.mode == GPURIR_POLY ? (poly ? GPURIR_POLY : GPURIR_FP32) : o.mode;
    const bool persistent = poly || use_persistent(((nISM + kTC - 1) / kTC) * M, o.split, d->num_sms);
    const int tile_len = poly ? kPolyTile : persistent ? kTCPersistent : kTC;
    A.nTiles = (int)((nISM + tile_len - 1) / tile_len);
    fill_common(A, fs, c, o.Tw);
    A.out = out;
    A.status = status_ptr(o, d);
    if ((st = setup_mode(d, o, fs, H, stream, A))) return st;
    A.poly_force2 = o.split == -2;
    A.poly_hook = o.split == -3 ? 2 : o.split == -5 ? 3 : 0;
    A.poly_gbz = A.poly_force2 || A.poly_hook == 3 || poly_two_word_for(room_sz, nISM, fs, c, o.Tw);
    // polyphase: the diffuse tail runs inside the ISM kernel when the envelope window (10 ms) fits the last
    // 1024-sample tile (and the call has GPURIR_FUSE_MIN_PER_SM RIRs per SM: 0, measured faster at every size)
    const int win = (int)llround(0.010 * fs);
    fused_tail = poly && nISM < nS && win <= kPolyTile && M >= (long long)GPURIR_FUSE_MIN_PER_SM * d->num_sms &&
                 fuse_tail_enabled();
    if (fused_tail) {
      A.poly_tail = 1;
      A.tail_win = win;
      A.tail_nS = (int)nS;
      const double T60 = sabine(room_sz, beta);
      A.tail_kappa_fs = isinf(T60) ? 0.f : (float)(6.0 * log(10.0) / T60 / fs);  // Eq. 8, reading C14
      A.tail_seed = o.seed;
      A.tail_rir_base = o.rir_index_base;
    }
    long long nclusters = (long long)A.nTiles * M;
    SlotGuard slab_guard;  // records the slab slot's event after the launch below (end of this scope)
    if (poly && (st = set_poly_slab(d, A, nclusters, o.split, stream, slab_guard))) return st;
    if (o.ev_ism[0]) cudaEventRecord((cudaEvent_t)o.ev_ism[0], stream);
    cudaError_t e;
    if (poly) {
      e = launch_ism_poly(A, nclusters, take_counter(d), d->num_sms, o.split, stream);
    } else if (persistent) {
      e = launch_ism_ws(A, kmode, nclusters, take_counter(d), d->num_sms, stream);
    } else {
      int split = auto_split(nclusters, o.split);
      e = launch_ism(A, kmode, split, nclusters, stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "launch_ism");
    if (o.ev_ism[1]) cudaEventRecord((cudaEvent_t)o.ev_ism[1], stream);
  }
  if (nISM < nS && fused_tail) {  // the tail was written by the polyphase kernel: the events bracket nothing
    if (o.ev_tail[0]) cudaEventRecord((cudaEvent_t)o.ev_tail[0], stream);
    if (o.ev_tail[1]) cudaEventRecord((cudaEvent_t)o.ev_tail[1], stream);
  } else if (nISM < nS) {
    TailArgs T;
    memset(&T, 0, sizeof(T));
    T.pos_src = pos_src; T.pos_rcv = pos_rcv; T.M_rcv = M_rcv; T.M = (int)M;
    T.nISM = (int)nISM; T.nS = (int)nS; T.row_stride = nS;
    double T60 = sabine(room_sz, beta);
    T.kappa_fs = isinf(T60) ? 0.f : (float)(6.0 * log(10.0) / T60 / fs);  // Eq. 8, reading C14
    T.rir_base = o.rir_index_base;
    T.fs_over_c = fs / c;
    T.win = (int)llround(0.010 * fs);
    T.seed = o.seed;
    T.out = out;
    long long groups = (nS + 3) / 4 - nISM / 4;
    // One warp per tail chunk.  Large calls: one chunk (up to kTailChunk samples) per RIR — splitting cfg3's
    // 8400-sample tails over 3 warps measured 10 % slower (the per-warp envelope reduction dominates).  Calls
    // with fewer RIRs than resident warps: split each tail (>= 64 Philox blocks per warp) so that a single
    // RIR's tail is not one warp's serial loop (latency of small calls, configs 1, 2 and 4).
    const long long slots = (long long)d->num_sms * 48;  // resident tail warps (6 CTAs x 8 warps per SM)
    long long nch = 1;
    if (M < slots) nch = std::max(1LL, std::min((slots + M - 1) / M, groups / 64));
    nch = std::max(nch, (groups + kTailChunk / 4 - 1) / (kTailChunk / 4));
    T.chunks_per_rir = (int)nch;
    T.chunk_quads = (int)((groups + nch - 1) / nch);
    if (o.ev_tail[0]) cudaEventRecord((cudaEvent_t)o.ev_tail[0], stream);
    cudaError_t e = launch_tail(T, (long long)T.chunks_per_rir * M, stream);
    if (e != cudaSuccess) return cuda_fail(e, "launch_tail");
    if (o.ev_tail[1]) cudaEventRecord((cudaEvent_t)o.ev_tail[1], stream);
  }
  return finish(o, stream, d);
}

int gpurir_simulate_rir_host(const float room_sz[3], const float beta[6], const float* pos_src, int M_src,
                             const float* orV_src, int spkr_pattern, const float* pos_rcv, int M_rcv,
                             const float* orV_rcv, int mic_pattern, const int nb_img[3], double Tdiff, double Tmax,
                             double fs, double c, float* out, const gpurir_opts* opts) {
  gpurir_opts o;
  if (opts) o = *opts; else gpurir_opts_default(&o);
  if (M_src <= 0 || M_rcv <= 0 || !pos_src || !pos_rcv || !out) return GPURIR_EINVAL;
  if (!(fs > 0) || !(c > 0) || !(Tmax > 0) || !(Tdiff >= 0)) return GPURIR_EINVAL;
  if (mic_pattern != GPURIR_OMNI && !orV_rcv) return GPURIR_EINVAL;
  if (spkr_pattern < 0 || spkr_pattern > 4 || (spkr_pattern != GPURIR_OMNI && !orV_src)) return GPURIR_EINVAL;
  const long long nS = gpurir_nsamples(Tmax, fs);
  if (nS > (1LL << 30) || (long long)M_src * M_rcv > (1LL << 30)) return GPURIR_EINVAL;
  int st = GPURIR_OK;
  DeviceState* d = device_state(&st);
  if (!d) return st;
  std::lock_guard<std::mutex> hk(d->host_mu);
  cudaError_t e = cudaSuccess;
  if (!d->copy_stream) {
    e = cudaStreamCreateWithFlags(&d->copy_stream, cudaStreamNonBlocking);
    for (int b = 0; b < 4 && e == cudaSuccess; b++) e = cudaEventCreateWithFlags(&d->host_ev[b], cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "host call streams");
  }
  cudaStream_t cs = (cudaStream_t)o.stream, xs = d->copy_stream;
  cudaEvent_t* computed = d->host_ev;
  cudaEvent_t* copied = d->host_ev + 2;
  // chunks of whole output rows: a receiver range of one source, or whole sources when M_rcv is small
  const long long chunk_target = std::max<long long>(kHostChunkMin, ((long long)M_src * M_rcv + 7) / 8);
  const bool by_rcv = M_rcv >= chunk_target;
  const int rcv_chunk = by_rcv ? (int)chunk_target : M_rcv;
  const int src_chunk = by_rcv ? 1 : (int)std::max<long long>(1, chunk_target / M_rcv);
  const size_t rows = (size_t)src_chunk * rcv_chunk;
  const size_t in_bytes = ((size_t)M_src * (orV_src ? 6 : 3) + (size_t)M_rcv * (orV_rcv ? 6 : 3)) * sizeof(float);
  const size_t in_pad = (in_bytes + 255) & ~(size_t)255;
  const size_t need = in_pad + 2 * rows * (size_t)nS * sizeof(float);
  if (need > d->host_scratch_bytes) {  // grow-only: later calls of this size reuse it (no allocator traffic)
    if (d->host_scratch) {
      cudaFree(d->host_scratch);  // private to host calls, which return only after their work has finished
      d->host_scratch = nullptr;
      d->host_scratch_bytes = 0;
    }
    e = cudaMalloc((void**)&d->host_scratch, need);
    if (e != cudaSuccess) { cudaGetLastError(); d->host_scratch = nullptr; return GPURIR_ENOMEM; }
    d->host_scratch_bytes = need;
  }
  char* scratch = d->host_scratch;
  float* d_src = reinterpret_cast<float*>(scratch);
  float* d_ors = orV_src ? d_src + 3 * (size_t)M_src : nullptr;
  float* d_rcv = d_src + (orV_src ? 6 : 3) * (size_t)M_src;
  float* d_orv = orV_rcv ? d_rcv + 3 * (size_t)M_rcv : nullptr;
  float* d_buf[2];
  d_buf[0] = reinterpret_cast<float*>(scratch + in_pad);
  d_buf[1] = d_buf[0] + rows * (size_t)nS;
  e = cudaMemcpyAsync(d_src, pos_src, 3 * sizeof(float) * M_src, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && orV_src)
    e = cudaMemcpyAsync(d_ors, orV_src, 3 * sizeof(float) * M_src, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_rcv, pos_rcv, 3 * sizeof(float) * M_rcv, cudaMemcpyHostToDevice, cs);
  if (e == cudaSuccess && orV_rcv)
    e = cudaMemcpyAsync(d_orv, orV_rcv, 3 * sizeof(float) * M_rcv, cudaMemcpyHostToDevice, cs);
  if (e != cudaSuccess) st = cuda_fail(e, "host call setup");
  gpurir_opts sub = o;
  sub.stream = cs;
  sub.flags &= ~GPURIR_FLAG_SYNC;
  long long k = 0;
  for (int s0 = 0; s0 < M_src && st == GPURIR_OK; s0 += src_chunk) {
    const int ns = std::min(src_chunk, M_src - s0);
    for (int r0 = 0; r0 < M_rcv && st == GPURIR_OK; r0 += rcv_chunk) {
      const int nr = std::min(rcv_chunk, M_rcv - r0);
      const int b = (int)(k & 1);
      if (k >= 2) cudaStreamWaitEvent(cs, copied[b], 0);  // d_buf[b] is free once chunk k-2 is on the host
      const long long row0 = (long long)s0 * M_rcv + r0;  // global index of the chunk's first RIR
      sub.rir_index_base = o.rir_index_base + (uint64_t)row0;
      st = gpurir_simulate_rir_dir(room_sz, beta, d_src + 3 * (size_t)s0, ns, d_ors ? d_ors + 3 * (size_t)s0 : nullptr,
                                   spkr_pattern, d_rcv + 3 * (size_t)r0, nr, d_orv ? d_orv + 3 * (size_t)r0 : nullptr,
                                   mic_pattern, nb_img, Tdiff, Tmax, fs, c, d_buf[b], &sub);
      if (st != GPURIR_OK) break;
      e = cudaEventRecord(computed[b], cs);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(xs, computed[b], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(out + row0 * nS, d_buf[b], (size_t)ns * nr * nS * sizeof(float), cudaMemcpyDeviceToHost, xs);
      if (e == cudaSuccess) e = cudaEventRecord(copied[b], xs);
      if (e != cudaSuccess) st = cuda_fail(e, "host call chunk");
      k++;
    }
  }
  // the caller's stream resumes after the last copy; the call returns when out is filled
  for (int b = 0; b < 2; b++)
    if (k > b) cudaStreamWaitEvent(cs, copied[b], 0);
  e = cudaStreamSynchronize(cs);
  if (st != GPURIR_OK) return st;
  if (e != cudaSuccess) return cuda_fail(e, "host call sync");
  gpurir_opts fin = o;
  fin.flags |= GPURIR_FLAG_SYNC;
  return finish(fin, cs, d);
}

long long gpurir_batch_extent(int n_rooms, const gpurir_room* rooms, double fs) {
  if (n_rooms < 0 || (n_rooms > 0 && !rooms) || !(fs > 0)) return -1;
  long long need = 0;
  for (int i = 0; i < n_rooms; i++) need = std::max(need, rooms[i].out_offset + gpurir_nsamples(rooms[i].Tmax, fs));
  return need;
}

size_t gpurir_workspace_bytes(int n_rooms, const gpurir_room* rooms, double fs, double c, const gpurir_opts* opts) {
  gpurir_opts o;
  if (opts) o = *opts; else gpurir_opts_default(&o);
  if (!(o.Tw > 0)) o.Tw = 4e-3;
  int st = GPURIR_OK;
  DeviceState* d = device_state(&st);
  if (!d) return 0;
  thread_local BatchPlan plan;
  BatchPlan& P = plan;
  P.reset();
  if (plan_batch(n_rooms, rooms, fs, c, o, d->num_sms, P) != GPURIR_OK) return 0;
  return P.bytes;
}

int gpurir_simulate_rir_batch(int n_rooms, const gpurir_room* rooms, double fs, double c, float* out,
                              const gpurir_opts* opts) {
  gpurir_opts o;
  if (opts) o = *opts; else gpurir_opts_default(&o);
  if (!(o.Tw > 0)) o.Tw = 4e-3;
  if (o.lut_Q <= 0) o.lut_Q = 16;
  if (!out) return GPURIR_EINVAL;
  int st = GPURIR_OK;
  DeviceState* d = device_state(&st);
  if (!d) return st;
  thread_local BatchPlan plan;
  BatchPlan& P = plan;
  P.reset();
  const double t_start = plan_timing() ? now_ms() : 0.0;
  if ((st = plan_batch(n_rooms, rooms, fs, c, o, d->num_sms, P))) return st;
  const double t_plan = plan_timing() ? now_ms() : 0.0;
  const double H = o.Tw * fs / 2.0;
  cudaStream_t stream = (cudaStream_t)o.stream;
  if (o.workspace && o.workspace_bytes < P.bytes) return GPURIR_EINVAL;
  if (o.workspace && (reinterpret_cast<uintptr_t>(o.workspace) & 255)) return GPURIR_EINVAL;

  // device workspace: the caller's, else the stream-ordered pool
  unsigned char* ws = reinterpret_cast<unsigned char*>(o.workspace);
  cudaError_t e = cudaSuccess;
  if (!ws) {
    e = cudaMallocAsync((void**)&ws, P.bytes, stream);
    if (e != cudaSuccess) { cudaGetLastError(); return GPURIR_ENOMEM; }
  }
  auto release = [&] {
    if (!o.workspace) cudaFreeAsync(ws, stream);
  };
  const double t_alloc = plan_timing() ? now_ms() : 0.0;
  BatchJob* djobs = reinterpret_cast<BatchJob*>(ws);
  int2* dtiles = reinterpret_cast<int2*>(ws + P.off_tiles);
  int2* dchunks = reinterpret_cast<int2*>(ws + P.off_chunks);
  const size_t bj = P.jobs.size() * sizeof(BatchJob), bt = P.tiles.size() * sizeof(int2),
               bc = P.chunks.size() * sizeof(int2);
  {
    // upload through a pinned staging slot: an asynchronous copy, no host synchronisation (the slot's previous
    // copy is waited for only if it has not executed yet, i.e. two batch calls are still queued before it)
    std::lock_guard<std::mutex> lk(d->stage_mu);
    const unsigned k = d->stage_next++ & 1u;
    if (!d->stage_done[k]) {
      e = cudaEventCreateWithFlags(&d->stage_done[k], cudaEventDisableTiming);
      if (e != cudaSuccess) { release(); return cuda_fail(e, "batch staging event"); }
    } else {
      e = cudaEventSynchronize(d->stage_done[k]);
      if (e != cudaSuccess) { release(); return cuda_fail(e, "batch staging wait"); }
    }
    if (d->stage_bytes[k] < P.bytes) {
      if (d->stage_host[k]) cudaFreeHost(d->stage_host[k]);
      d->stage_host[k] = nullptr;
      d->stage_bytes[k] = 0;
      const size_t want = P.bytes + P.bytes / 4;
      e = cudaMallocHost((void**)&d->stage_host[k], want);
      if (e != cudaSuccess) { cudaGetLastError(); release(); return GPURIR_ENOMEM; }
      d->stage_bytes[k] = want;
    }
    char* h = d->stage_host[k];
    memcpy(h, P.jobs.data(), bj);
    if (bt) memcpy(h + P.off_tiles, P.tiles.data(), bt);
    if (bc) memcpy(h + P.off_chunks, P.chunks.data(), bc);
    e = cudaMemcpyAsync(ws, h, P.off_chunks + bc, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaEventRecord(d->stage_done[k], stream);
    if (e != cudaSuccess) { release(); return cuda_fail(e, "batch upload"); }
  }
  const double t_stage = plan_timing() ? now_ms() : 0.0;
  struct TimingPrint {  // at return: the launch phase ends with the call
    double t0, t1, t2, t3;
    int n;
    ~TimingPrint() {
      if (!plan_timing()) return;
      fprintf(stderr, "gpurir batch %d rooms: plan %.2f ms, workspace %.2f ms, staging %.2f ms, launch %.2f ms\n", n,
              t1 - t0, t2 - t1, t3 - t2, now_ms() - t3);
    }
  } timing_print{t_start, t_plan, t_alloc, t_stage, n_rooms};

  if (!P.tiles.empty()) {
    IsmArgs A;
    memset(&A, 0, sizeof(A));
    A.jobs = djobs; A.tiles = dtiles;
    fill_common(A, fs, c, o.Tw);
    A.out = out;
    A.status = status_ptr(o, d);
    if ((st = setup_mode(d, o, fs, H, stream, A))) { release(); return st; }
    A.poly_force2 = o.split == -2;
    A.poly_hook = o.split == -3 ? 2 : o.split == -5 ? 3 : 0;
    A.poly_gbz = A.poly_force2 || A.poly_hook == 3 || P.any_two_word;
    if (P.fused) {
      A.poly_tail = 1;
      A.tail_win = (int)llround(0.010 * fs);
      A.tail_seed = o.seed;
    }
    const long long nw = (long long)P.tiles.size();
    SlotGuard slab_guard;
    if (P.poly && (st = set_poly_slab(d, A, nw, o.split, stream, slab_guard))) { release(); return st; }
    if (o.ev_ism[0]) cudaEventRecord((cudaEvent_t)o.ev_ism[0], stream);
    if (P.poly) e = launch_ism_poly(A, nw, take_counter(d), d->num_sms, o.split, stream);
    else if (P.persistent) e = launch_ism_ws(A, P.kmode, nw, take_counter(d), d->num_sms, stream);
    else e = launch_ism(A, P.kmode, auto_split(nw, o.split), nw, stream);
    if (e != cudaSuccess) { release(); return cuda_fail(e, "launch_ism(batch)"); }
    if (o.ev_ism[1]) cudaEventRecord((cudaEvent_t)o.ev_ism[1], stream);
  }
  if (o.ev_tail[0]) cudaEventRecord((cudaEvent_t)o.ev_tail[0], stream);
  if (!P.chunks.empty()) {
    TailArgs T;
    memset(&T, 0, sizeof(T));
    T.jobs = djobs; T.chunks = dchunks;
    T.fs_over_c = fs / c;
    T.win = (int)llround(0.010 * fs);
    T.seed = o.seed;
    T.out = out;
    T.chunk_quads = kTailChunk / 4;
    e = launch_tail(T, (long long)P.chunks.size(), stream);
    if (e != cudaSuccess) { release(); return cuda_fail(e, "launch_tail(batch)"); }
  }
  if (o.ev_tail[1]) cudaEventRecord((cudaEvent_t)o.ev_tail[1], stream);
  release();
  return finish(o, stream, d);
}

int gpurir_simulate_trajectory(const float* signal, long long n_sig, const float* rirs, int n_points, int n_mics,
                               long long rir_len, float* out, const gpurir_opts* opts) {
  gpurir_opts o;
  if (opts) o = *opts; else gpurir_opts_default(&o);
  if (!signal || !rirs || !out || n_sig <= 0 || n_points <= 0 || n_mics <= 0 || rir_len <= 0) return GPURIR_EINVAL;
  if (n_sig < n_points || n_mics > 65535 || n_sig + rir_len > (1LL << 40)) return GPURIR_EINVAL;
  cudaStream_t stream = (cudaStream_t)o.stream;
  int st = GPURIR_OK;
  DeviceState* d = device_state(&st);
  if (!d) return st;
  cudaError_t e;
  // the tcgen05 kernel (traj_tc_kernel.cu) when the RIR bank allows 16-B loads; opts.split = -1 forces the
  // CUDA-core kernel (traj_kernel.cu), split > 0 the tensor-core kernel's K split (test hooks)
  const size_t pw = o.split >= 0 && traj_tc_supported(rirs, rir_len)
                        ? traj_tc_part_words(signal, n_sig, rirs, n_points, n_mics, rir_len, d->num_sms, o.split)
                        : 0;
  SlotGuard part_guard;  // records the partials slot's event after the launch (end of this function)
  if (pw > 0) {
    float* part = nullptr;
    {
      unsigned k;
      {
        std::lock_guard<std::mutex> lk(g_mu);
        k = d->next_traj++ % 2;
      }
      part_guard.take(d->slot_mu, &d->traj_ev[k], stream);
      if (int st = grow_ring(d->traj_part, d->traj_part_words, 2, pw, part_guard.capturing, "traj partials"))
        return st;
      part = d->traj_part[k];
    }
    e = launch_traj_tc(signal, n_sig, rirs, n_points, n_mics, rir_len, out, part, d->num_sms, o.split, stream);
  } else {
    e = launch_traj(signal, n_sig, rirs, n_points, n_mics, rir_len, out, stream);
  }
  if (e != cudaSuccess) return cuda_fail(e, "launch_traj");
  return finish(o, stream, d);
}

int gpurir_image_params(const float room_sz[3], const float beta[6], const float src[3], const float rcv[3],
                        const float orv[3], int mic_pattern, const float ors[3], int spkr_pattern,
                        const int nb_img[3], double fs, double c, double* x_out, float* A_out, void* stream_) {
  int st = validate_room(room_sz, beta, nb_img, mic_pattern);
  if (st) return st;
  if (spkr_pattern < 0 || spkr_pattern > 4 || (spkr_pattern != GPURIR_OMNI && !ors)) return GPURIR_EINVAL;
  if (!(fs > 0) || !(c > 0) || !x_out || !A_out || !src || !rcv) return GPURIR_EINVAL;
  DeviceState* d = device_state(&st);
  if (!d) return st;
  cudaStream_t stream = (cudaStream_t)stream_;
  BatchJob J;
  memset(&J, 0, sizeof(J));
  for (int a = 0; a < 3; a++) {
    J.L[a] = room_sz[a]; J.src[a] = src[a]; J.rcv[a] = rcv[a]; J.orv[a] = orv ? orv[a] : 0.f; J.nb[a] = nb_img[a];
  }
  for (int w = 0; w < 6; w++) J.beta[w] = beta[w];
  beta_logs(beta, J.lb, &J.neg, &J.zero);
  J.pattern = mic_pattern;
  if (mic_pattern != GPURIR_OMNI && !orv) return GPURIR_EINVAL;
  for (int a = 0; a < 3; a++) J.ors[a] = ors ? ors[a] : 0.f;
  J.spkr_pattern = spkr_pattern;
  BatchJob* dj = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dj, sizeof(BatchJob), stream);
  if (e != cudaSuccess) return GPURIR_ENOMEM;
  e = cudaMemcpyAsync(dj, &J, sizeof(J), cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "image_params upload");
  IsmArgs A;
  memset(&A, 0, sizeof(A));
  A.jobs = dj;
  fill_common(A, fs, c, 4e-3);
  A.status = d->status;
  long long N = (long long)nb_img[0] * nb_img[1] * nb_img[2];
  e = launch_image_params(A, x_out, A_out, N, stream);
  if (e != cudaSuccess) return cuda_fail(e, "launch_image_params");
  cudaFreeAsync(dj, stream);
  gpurir_opts o;
  gpurir_opts_default(&o);
  o.flags = GPURIR_FLAG_SYNC;
  return finish(o, stream, d);
}

int gpurir_device_status(int reset) {
  int st = GPURIR_OK;
  DeviceState* d = device_state(&st);
  if (!d) return st;
  int s = 0;
  cudaError_t e = cudaMemcpy(&s, d->status, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "status");
  if (reset) cudaMemset(d->status, 0, sizeof(int));
  if (!s) return GPURIR_OK;
  return status_code(s);
}

const char* gpurir_strerror(int status) {
  switch (status) {
    case GPURIR_OK: return "ok";
    case GPURIR_EINVAL: return "invalid argument";
    case GPURIR_EDEGENERATE: return "degenerate geometry (image source on a receiver)";
    case GPURIR_EINFEASIBLE: return "infeasible target T60";
    case GPURIR_ENOMEM: return "out of device memory";
    case GPURIR_ECUDA: return "CUDA error";
    case GPURIR_ECAPACITY: return "capacity: more than 2^17 images on one sample of a polyphase tile";
  }
  return "unknown status";
}

const char* gpurir_last_cuda_error(void) { return g_cuda_err; }

#ifdef GPURIR_VARIANT  // A/B builds (tools/build_variant.sh); bench.py refuses to time them without --ab-lib
const char* gpurir_version(void) { return "gpurir-b200 0.2.0 (sm_100a) variant:" GPURIR_VARIANT; }
#else
const char* gpurir_version(void) { return "gpurir-b200 0.2.0 (sm_100a)"; }
#endif

}  // extern "C"

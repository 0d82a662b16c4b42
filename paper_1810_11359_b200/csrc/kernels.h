// kernels.h — host <-> device argument blocks and launchers of libgpurir.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace gpurir {

constexpr int kPolyMaxItems = 320;  // polyphase calls whose work items' output ranges may be split (<= 2 items per SM)
constexpr int kPolyMaxSubItems = 320;  // the split plan's (item, sub-range) entries: at most one wave
static_assert(kPolyMaxItems < 1024 && kPolyMaxSubItems <= 65535, "plan map: item | sub << 10 | log2(nsub) << 12");
constexpr int kPolyClusterMaxItems = 32;  // polyphase calls of at most this many (tile, RIR) items run cluster items

// One RIR of a multi-room batch (device copy built by the host planner).
struct alignas(16) BatchJob {
  float L[3];
  float beta[6];
  float src[3];
  float rcv[3];
  float orv[3];
  int pattern;
  int nb[3];
  int nISM;             // ISM samples of this RIR
  int nS;               // total samples of this RIR
  long long out_offset; // element offset of the RIR row in the output
  float kappa_fs;       // kappa / fs (1/sample) of the Sabine envelope (Eq. 8, C14)
  unsigned long long rir_global;  // tail RNG stream id (C16)
  float lb[6];          // log2 |beta_w| (0 where beta_w == 0), precomputed on the host
  unsigned neg, zero;   // bit w: beta_w < 0 / beta_w == 0
  float ors[3];         // source orientation (f3, reading R10; ignored for an omni source)
  int spkr_pattern;     // source polar pattern (gpurir_pattern)
  double geo[5];        // host-computed reciprocals for the polyphase tile setup: 1/L[0..2] (m^-1), 1/V_s (samples^-3),
                        // 1/L_min,s (samples^-1) — see IsmArgs::poly_geo
};

struct IsmArgs {
  // single-room call (jobs == nullptr)
  float L[3];
  float beta[6];
  float lb[6];           // log2 |beta_w| (0 where beta_w == 0), precomputed on the host
  unsigned neg, zero;    // bit w: beta_w < 0 / beta_w == 0
  int nb[3];
  int pattern;
  const float* pos_src;
  const float* pos_rcv;
  const float* orv;
  const float* ors;      // source orientations [M_src][3] or nullptr (omni source; f3)
  int spkr_pattern;
  int M_src, M_rcv, M;
  int nISM;
  long long row_stride;  // nSamples
  int nTiles;
  // batch call
  const BatchJob* jobs;
  const int2* tiles;     // per cluster: (job, tile)
  // common
  double fs_over_c, c_over_fs;
  // polyphase tile setup without divisions (single-room calls; batch jobs carry their own BatchJob::geo):
  // 1/L[0..2], 1/V_s, 1/L_min,s as in BatchJob::geo, and 1/M, 1/M_rcv for the work-item decode (exact, fix-up)
  double poly_geo[5];
  double invM, invMrcv;
  float H, invH;         // half window (samples) and 1/H
  int nbw;               // delay bins touching one warp sub-tile
  // exact power-of-two scaling of the tap argument: Hs = 2^ceil(log2 H),
  // v = u / Hs, rho = H / Hs; window polynomial in sigma = v^2 - rho^2 with coefficients wb[i]
  float invHs;           // 1 / Hs
  float rho2;            // rho^2
  float wb[3];           // b_i / rho^(2i+2)
  float wa[4];           // the same window as a polynomial in u = 1 + sigma (sat-clamped form), wa[0] = -sum
  float urho;            // 1 - rho^2
  float hc[3];           // fp16 mode: Eq. 11 coefficients of x^2, x^4, x^6 divided by rho^2, rho^4, rho^6
  float x2clamp;         // fp16 mode: rho^2 / 4
  float* out;
  int* status;
  // LUT mode
  const float2* lut;     // phase-major rows [Q][cols] of (T[n+1], T[n]-T[n+1])
  int lut_rows, lut_cols, lut_joff, lutQ;
  // texture-LUT mode: the Eq. 9 table T[n], n = -half..half, in a 1-D CUDA array
  // sampled with hardware linear filtering; a tap at offset u = k - x samples reads coordinate u Q + tex_off
  unsigned long long tex;  // cudaTextureObject_t
  float texQ, tex_off;     // Q and half + 0.5 (texel centres)
  // polyphase mode (reading R11): delta'(m - phi) = sum_d P[m - mlo][d] T_d(2 phi - 1), m = mlo .. mlo + ntaps - 1
  // FIR tables (reading R13, abi.cu poly_fir_tables): far [2][ntaps][2], near [2][nn][2] (taps nmi0 ..), Q [8][8]
  const float* poly_P;
  int poly_ntaps, poly_mlo;
  int poly_nmi0, poly_nn;
  // constants of the image walk read as parameter-bank operands (literals would be re-materialised every image at
  // the 64-register cap): 2^52 + 2^31 (the int -> double trick's bias) and -1
  double poly_i2d_bias;
  float poly_m1;
  int poly_gbz;            // some tile of the call starts in the two-word scheme: zero the fine plane Gb per tile
  int poly_gb;             // set by the launcher: the fine plane Gb is allocated (two-word tiles, guard's last rung)
  int poly_force2;         // test hook (opts.split == -2): every tile uses the two-word scheme
  int poly_hook;           // test hooks of the count guard (capacity 4 images per position): 2 (split -3) on the
                           // first pass (-> redo in two words, or the capacity status without the fine plane);
                           // 3 (split -5) two words on every tile (-> the capacity status)
  // polyphase single-room calls: the diffuse tail fused into the kernel — the CTA that finishes a RIR's last
  // (end-aligned) ISM tile, which holds the whole envelope window, writes that RIR's tail (tail_common.cuh)
  int poly_tail;
  int tail_win, tail_nS;
  float tail_kappa_fs;
  unsigned long long tail_seed, tail_rir_base;
  // polyphase small calls (thread-block cluster items): the ranks' integer planes meet through global memory (L2
  // moves several times the ~20 B/clk per SM of distributed shared memory): per CTA a slab of poly_slab_planes x
  // poly_slab_w words, then per cluster kPolyD x poly_slab_w fp32 totals (scratch owned by the library)
  unsigned* poly_slab;
  int poly_slab_w;
  // polyphase small single-room calls: a heavy tile's OUTPUT range split into 2 or 4 sub-ranges, each a cluster
  // item of its own (the tile's fixed-point format is kept, so its G and every output are the same bits); item i
  // (= tile x RIR work item) owns clusters [poly_first[i], poly_first[i + 1]); poly_nitems = 0: one cluster each
  int poly_nitems;
  unsigned short poly_first[kPolyMaxItems + 1];
  // the same plan per cluster (cluster items) or per queue entry (persistent CTAs): item | sub << 10 | log2(nsub) << 12
  unsigned short poly_cmap[kPolyMaxSubItems];
};

struct TailArgs {
  // single-room call (jobs == nullptr)
  const float* pos_src;
  const float* pos_rcv;
  int M_rcv, M;
  int nISM, nS;
  long long row_stride;
  float kappa_fs;
  unsigned long long rir_base;
  // batch
  const BatchJob* jobs;
  const int2* chunks;    // per CTA: (job, chunk)
  // common
  double fs_over_c;
  int win;               // estimation window length in samples, round(0.010 fs) (C15)
  unsigned long long seed;
  float* out;
  int chunks_per_rir;
  int chunk_quads;       // Philox blocks (4 samples) per warp item
};

size_t ism_smem_bytes(int mode, int lut_rows, int lut_cols);
cudaError_t launch_ism(const IsmArgs& A, int mode, int split, long long nclusters, cudaStream_t stream);
cudaError_t launch_image_params(const IsmArgs& A, double* x_out, float* A_out, long long N, cudaStream_t stream);
size_t ism_ws_smem_bytes(int mode, int lut_rows, int lut_cols);
cudaError_t launch_ism_ws(const IsmArgs& A, int mode, long long n_work, int* counter, int num_sms,
                          cudaStream_t stream);
size_t ism_poly_smem_bytes(int ntaps, bool two_word);
cudaError_t launch_ism_poly(const IsmArgs& A, long long n_work, int* counter, int num_sms, int split,
                            cudaStream_t stream);
int ism_poly_cluster_size(long long n_work, int num_sms, int split, int ntaps, bool two_word,
                          int* threads);  // cluster size S of a call's items (0: persistent CTAs)
size_t ism_poly_slab_words(long long n_work, int S, int ntaps, int num_sms);  // cluster items' L2 exchange scratch
cudaError_t launch_tail(const TailArgs& A, long long n_items, cudaStream_t stream);  // one warp per item

cudaError_t launch_traj(const float* sig, long long n_sig, const float* rirs, int n_points, int n_mics, long long L,
                        float* out, cudaStream_t stream);
// tensor-core trajectory filter (traj_tc_kernel.cu): RIR length a multiple of 4 and a 16-B aligned RIR bank
bool traj_tc_supported(const float* rirs, long long L);
size_t traj_tc_part_words(const float* sig, long long n_sig, const float* rirs, int n_points, int n_mics, long long L,
                          int num_sms, int force);  // K-split partial scratch (0: the tensor-core kernel cannot run)
cudaError_t launch_traj_tc(const float* sig, long long n_sig, const float* rirs, int n_points, int n_mics, long long L,
                           float* out, float* partial, int num_sms, int force, cudaStream_t stream);

constexpr int kTailThreads = 256;
constexpr int kTailChunk = kTailThreads * 64;  // samples per tail CTA (up to 16 Philox blocks per thread)

}  // namespace gpurir

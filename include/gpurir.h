/*
 * gpurir.h — C ABI of libgpurir.so, the B200 (sm_100a) Image Source Method
 * room-impulse-response engine (the hot path of gpuRIR, arXiv 1810.11359).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; readings "C<k>" are
 * listed in DESIGN.md §Readings.
 *
 * Conventions (all entry points):
 *   - extern "C", no exceptions; every call returns a gpurir_status (0 = OK)
 *     unless documented otherwise.
 *   - Arrays documented "device" are caller-owned CUDA device pointers on the
 *     calling thread's current device; "host" arrays are read before return.
 *   - Output buffers are written in place and never allocated or freed by the
 *     library.  Calls are stream-ordered on opts->stream and return without a
 *     device synchronisation unless GPURIR_FLAG_SYNC is set.
 *   - There is no global mutable state (the paper's global LUT / mixed-
 *     precision switches, become the per-call opts->mode).  Per device
 *     the library keeps a status word, a LUT cache and a ring of 256 work-
 *     queue counters, so up to 256 calls may be in flight concurrently on
 *     different streams of one device; the scratch of small polyphase calls
 *     (4 slots) and of the trajectory filter's partial sums (2 slots) is
 *     reused in stream order (an event per slot), so more concurrent calls
 *     than slots wait for the slot on the device, not on the host.  A call
 *     captured into a CUDA graph takes its slot at capture time; replays of
 *     one graph are ordered by their stream, concurrent replays of several
 *     graphs that captured the same slot are not.  Scratch grows only in an
 *     eager call (growing synchronises the device), so make one eager call of
 *     a size before capturing it; after that, gpurir_simulate_rir(_dir) and
 *     gpurir_simulate_trajectory are capturable (no host synchronisation,
 *     allocation or pageable copy on their path; tested for configs 1 and 2).
 *   - Validation runs on the host before any launch.  Conditions that can
 *     only be seen on the device (a zero orientation vector, an image source
 *     coinciding with a receiver) raise a per-device status word that is
 *     returned by the call when GPURIR_FLAG_SYNC is set, and otherwise by the
 *     next gpurir_device_status() call.
 */
#ifndef GPURIR_H
#define GPURIR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GPURIR_OK = 0,
  GPURIR_EINVAL = 1,       /* bad argument: sizes, |beta| > 1, pattern, times, zero orientation */
  GPURIR_EDEGENERATE = 2,  /* an image source coincides with a receiver, d_n = 0 */
  GPURIR_EINFEASIBLE = 3,  /* Sabine target T60 below the room's minimum */
  GPURIR_ENOMEM = 4,       /* device allocation failed */
  GPURIR_ECUDA = 5,        /* CUDA runtime error; see gpurir_last_cuda_error() */
  GPURIR_ECAPACITY = 6     /* capacity: GPURIR_POLY found more images on one sample position of a tile
                              than its exact integer sums can hold (2^17 in the two-word format; 2^(31 - bits)
                              in the single-word one when the call's CTAs have no room for the two-word redo)
                              — reported instead of a wrapped sum; re-run with opts->split = -2 */
} gpurir_status;

/* Receiver polar patterns, g = a + (1 - a) cos(theta) (reading C4). */
typedef enum {
  GPURIR_OMNI = 0,          /* a = 1    */
  GPURIR_SUBCARDIOID = 1,   /* a = 0.75 */
  GPURIR_CARDIOID = 2,      /* a = 0.5  */
  GPURIR_HYPERCARDIOID = 3, /* a = 0.25 */
  GPURIR_BIDIRECTIONAL = 4  /* a = 0    */
} gpurir_pattern;

/* Sinc evaluation mode (mutually exclusive). */
typedef enum {
  GPURIR_FP32 = 0, /* Eq. 6 evaluated in fp32 (the paper's "base" kernel)               */
  GPURIR_LUT = 1,  /* Eq. 9 windowed-sinc table, Q-times oversampled, linear interp.    */
  GPURIR_FP16 = 2, /* half2 tap arithmetic with the Eq. 10-12 style polynomials */
  GPURIR_LUT_TEX = 3, /* Eq. 9 table in texture memory, hardware linear interpolation (the paper's LUT
                        placement).  Any Q >= 1 with 2 ceil(Tw Q fs / 2) + 1 <= the
                        device's 1-D texture width (else EINVAL).  Interpolation weights have 8 fractional
                        bits (texture hardware); tolerance as GPURIR_LUT. */
  GPURIR_POLY = 4     /* Eq. 6 by its polyphase expansion (reading R11): every image adds
                        A_n T_d(2 phi_n - 1), d = 0..7, to the integer sample floor(x_n) (exact
                        fixed-point sums with a per-tile scale: one int32 word per channel, two for tiles
                        whose estimate of images per sample reaches 2^12; deterministic; a tile whose exact
                        per-sample image count reaches its word's capacity is redone wider, never wrapped —
                        GPURIR_ECAPACITY past 2^17), then an 8-channel FIR of 2H taps, whose
                        coefficients expand delta'(m - phi) in Chebyshev polynomials (max error 4.3e-7),
                        produces the RIR.  fp32 arithmetic; fp32 tolerance.  Requires Tw fs <= 1022.
                        Calls with fewer than 32 work items of 1024 samples (a lone RIR) run the direct
                        fp32 kernels instead, unless opts->split < 0 forces the polyphase kernel. */
} gpurir_mode;

#define GPURIR_FLAG_SYNC 1u /* synchronise the stream before returning and report device-side status */

typedef struct {
  int mode;                 /* gpurir_mode, default GPURIR_FP32                                    */
  double Tw;                /* Peterson window length in seconds, default 4e-3              */
  int lut_Q;                /* LUT oversampling factor Q, default 16                        */
  uint64_t seed;            /* diffuse-tail RNG key (Philox4x32-10, reading C16), default 0         */
  uint64_t rir_index_base;  /* global index of this call's first RIR (tail RNG stream id), default 0 */
  void* stream;             /* cudaStream_t to launch on; NULL = the legacy default stream          */
  int split;                /* CTAs cooperating on one time tile (thread-block cluster), 0 = auto;
                               < 0 forces the persistent kernel (fp32/LUT/fp16) or the polyphase kernel;
                               test hooks of GPURIR_POLY: -2 two-word scheme on every tile; -3 a count capacity
                               of 4 images per sample position on the first pass (exercises the overflow
                               guard: redo in two words, or GPURIR_ECAPACITY for a call launched without the
                               fine plane); -5 two-word tiles with that capacity (GPURIR_ECAPACITY) */
  unsigned flags;           /* GPURIR_FLAG_*                                                        */
  void* ev_ism[2];          /* optional cudaEvent_t pair recorded on `stream` around the ISM kernel  */
  void* ev_tail[2];         /* optional cudaEvent_t pair recorded around the diffuse-tail kernel     */
  void* workspace;          /* optional caller-owned device scratch of gpurir_simulate_rir_batch, 256-B
                               aligned, >= gpurir_workspace_bytes() bytes (EINVAL otherwise); NULL = the
                               stream-ordered pool (cudaMallocAsync / cudaFreeAsync on `stream`)          */
  size_t workspace_bytes;   /* its size                                                               */
  int* status;              /* optional caller-owned device int, zero-initialised: this call's status
                               word (device-side errors, read with GPURIR_FLAG_SYNC) instead of the
                               device's shared one — calls in flight on several streams stay separate    */
} gpurir_opts;

/* Fill *opts with the defaults above. */
void gpurir_opts_default(gpurir_opts* opts);

/*
 * gpurir_simulate_rir — RIRs of every (source, receiver) pair of one shoebox
 * room (Eqs. 1-6 for 0 <= t < Tdiff, diffuse tail Eqs. 7-8 / P:160 for
 * Tdiff <= t < Tmax).
 *   room_sz  host  float[3]   room size L (m), each > 0
 *   beta     host  float[6]   signed reflection coefficients (x0,x1,y0,y1,z0,z1), |beta| <= 1
 *   pos_src  device float[M_src][3]  source positions (m)
 *   pos_rcv  device float[M_rcv][3]  receiver positions (m)
 *   orV_rcv  device float[M_rcv][3]  receiver orientations (normalised on the device), may be NULL
 *                                    only when mic_pattern == GPURIR_OMNI
 *   nb_img   host  int[3]     images per axis N_x, N_y, N_z >= 1; lattice ceil(-N/2) <= n < ceil(N/2)
 *   Tdiff    ISM / diffuse switch time (s) >= 0; nISM = ceil(Tdiff fs) samples (reading C9)
 *            (at most 2^22 - 8192, the range the kernels' fp32 delay floor is exact on; else EINVAL)
 *   Tmax     RIR length (s) > 0; nSamples = ceil(Tmax fs) (C9); Tdiff >= Tmax means ISM only
 *   fs, c    sampling rate (Hz) and speed of sound (m/s), > 0
 *   out      device float[M_src][M_rcv][nSamples], caller-owned, row-major RIR r = m_src*M_rcv + m_rcv
 *   opts     NULL for defaults
 * Errors: EINVAL (host validation), EDEGENERATE / EINVAL from the device word
 * (see file header), ECUDA on a launch failure.
 */
int gpurir_simulate_rir(const float room_sz[3], const float beta[6], const float* pos_src, int M_src,
                        const float* pos_rcv, int M_rcv, const float* orV_rcv, int mic_pattern, const int nb_img[3],
                        double Tdiff, double Tmax, double fs, double c, float* out, const gpurir_opts* opts);

/*
 * gpurir_simulate_rir_dir — gpurir_simulate_rir with a directional source (reading
 * R10 of DESIGN.md; the paper models only the receiver pattern).
 *   orV_src      device float[M_src][3]  source orientations (normalised on the device), may be NULL only
 *                                       when spkr_pattern == GPURIR_OMNI
 *   spkr_pattern gpurir_pattern of every source: g_s = a + (1 - a) cos(theta_s), theta_s between the
 *                image's mirrored source orientation diag((-1)^n) o_s and p_r - p_n.
 * A_n = beta_n g_rcv g_src / (4 pi d_n).  Other arguments, layout and errors as gpurir_simulate_rir, which
 * is this call with an omni source (bit-identical results).
 */
int gpurir_simulate_rir_dir(const float room_sz[3], const float beta[6], const float* pos_src, int M_src,
                            const float* orV_src, int spkr_pattern, const float* pos_rcv, int M_rcv,
                            const float* orV_rcv, int mic_pattern, const int nb_img[3], double Tdiff, double Tmax,
                            double fs, double c, float* out, const gpurir_opts* opts);

/*
 * gpurir_simulate_rir_host — gpurir_simulate_rir_dir from HOST memory: the end-to-end call of a
 * dataset-generation loop (P:274's interface with the host<->device transfers inside; the paper's memcpy
 * step).  pos_src, orV_src, pos_rcv, orV_rcv and out have the layouts of gpurir_simulate_rir_dir
 * but are host pointers; page-locked (pinned) memory lets the copies run asynchronously, pageable memory
 * works but its copies are staged by the driver.  The call copies the positions to the device, then
 * computes the RIRs in chunks of whole rows (receiver ranges of one source, or groups of whole sources
 * when M_rcv is small) into two device buffers on opts->stream while a second stream copies the previous
 * chunk back into out, so the device->host transfer overlaps the kernels.  Every chunk keeps its global RIR
 * index (tail RNG stream, reading C16): the result equals one device call over all RIRs (bit-identical in
 * GPURIR_POLY mode, which is shard-invariant).  Device scratch (2 chunk outputs + positions) is a
 * grow-only per-device buffer kept for later calls; host calls on one device are serialised by a lock.
 * Synchronous: returns when out is filled (the status word is checked as with GPURIR_FLAG_SYNC).
 * opts->ev_ism / ev_tail are ignored.
 * Errors: as gpurir_simulate_rir_dir; ENOMEM when the scratch cannot be allocated; ECUDA on copy failure.
 */
int gpurir_simulate_rir_host(const float room_sz[3], const float beta[6], const float* pos_src, int M_src,
                             const float* orV_src, int spkr_pattern, const float* pos_rcv, int M_rcv,
                             const float* orV_rcv, int mic_pattern, const int nb_img[3], double Tdiff,
                             double Tmax, double fs, double c, float* out, const gpurir_opts* opts);

/* One independent room of a batch (config 5; a deviation from the paper's
 * same-room-only batching).  out_offset = element offset of this RIR's
 * row in the batch output buffer (ragged rows of ceil(Tmax fs) samples). */
typedef struct {
  float room_sz[3];
  float beta[6];
  float pos_src[3];
  float pos_rcv[3];
  float orV_rcv[3]; /* ignored for GPURIR_OMNI */
  int mic_pattern;
  int nb_img[3];
  double Tdiff;
  double Tmax;
  long long out_offset;
  float orV_src[3]; /* source orientation (f3), ignored for an omni source */
  int spkr_pattern; /* source gpurir_pattern (f3), GPURIR_OMNI = 0 for the paper's omni source */
  unsigned long long rir_index; /* this RIR's index in the whole job: its tail RNG stream is
                                   opts->rir_index_base + rir_index (reading C16), so a shard of rooms in any
                                   order reproduces the unsharded bits */
} gpurir_room;

/*
 * gpurir_simulate_rir_batch — one RIR per room for n_rooms independent rooms (config 5: dataset generation;
 * P:167 batches only RIRs of one room, the rooms of a dataset are as independent).
 *   rooms  host gpurir_room[n_rooms], read before return (planned on the host: a job table and a heavy-first
 *          tile list, uploaded through a pinned staging buffer by an asynchronous copy on opts->stream)
 *   out    device float buffer; room i writes out[rooms[i].out_offset + k], 0 <= k < ceil(Tmax_i fs)
 *   The tail RNG stream of room i is opts->rir_index_base + rooms[i].rir_index.
 * Stream-ordered: returns without synchronising (unless GPURIR_FLAG_SYNC); device scratch from
 * opts->workspace or the stream-ordered pool.  In GPURIR_POLY mode a room's RIR equals, bit for bit, the same
 * room simulated alone by gpurir_simulate_rir_dir (the tiles are end-aligned per room in both), and the
 * diffuse tail is written by the polyphase kernel (one launch per call).
 * Errors as gpurir_simulate_rir; ENOMEM if the workspace or the staging buffer cannot be allocated; EINVAL
 * for a caller workspace below gpurir_workspace_bytes() or not 256-B aligned.
 */
int gpurir_simulate_rir_batch(int n_rooms, const gpurir_room* rooms, double fs, double c, float* out,
                              const gpurir_opts* opts);

/* Device workspace (bytes) gpurir_simulate_rir_batch needs for these rooms and options (job table, tile and
 * chunk lists: about 100 B per room); 0 for invalid arguments.  Single-room calls need no workspace. */
size_t gpurir_workspace_bytes(int n_rooms, const gpurir_room* rooms, double fs, double c, const gpurir_opts* opts);

/* Elements of `out` a gpurir_simulate_rir_batch call with these rooms writes: max over i of
 * rooms[i].out_offset + ceil(Tmax_i fs) (reading C9, the same count as gpurir_nsamples).  Host only, no device
 * work; the caller sizes (or checks) its output buffer with it.  -1 for invalid arguments (n_rooms < 0, NULL
 * rooms with n_rooms > 0, fs <= 0). */
long long gpurir_batch_extent(int n_rooms, const gpurir_room* rooms, double fs);

/*
 * gpurir_simulate_trajectory — a moving source recorded by a microphone array (§3.4,
 * P:225-227; the trajectory-filtering function of P:276).
 *   signal  device float[n_sig]                      mono source signal
 *   rirs    device float[n_points][n_mics][rir_len]   RIR bank of every trajectory point (e.g. from
 *                                                     gpurir_simulate_rir with the points as sources)
 *   out     device float[n_mics][n_sig + rir_len - 1], caller-owned
 * The signal is split into n_points contiguous segments of floor(n_sig / n_points) samples (the last one
 * takes the remainder; reading R7); segment p is filtered by point p's RIRs and the filtered segments
 * are overlap-added: out[m][t] = sum_j signal[j] rirs[p(j)][m][t - j].  When rir_len is a multiple of 4 and
 * rirs 16-B aligned, the sum runs on the tensor cores (tcgen05, 3xTF32: fp32 accuracy, ~2^-22 per product): per
 * segment a banded Toeplitz matrix of the signal times windows of the RIRs, 128 outputs x 256 (block, mic)
 * columns per tile, K-split partial tiles summed in a fixed order; otherwise a direct fp32 convolution on the
 * CUDA cores.  Deterministic either way.  opts->split: 0 automatic, -1 forces the CUDA-core kernel, k > 0 the
 * tensor-core kernel with a K split of k (test hooks).  Device scratch for the K-split partials is owned by the
 * library (grow-only, allocated by the first call of a size).
 * Errors: EINVAL (n_sig < n_points, sizes <= 0, NULL pointers).
 */
int gpurir_simulate_trajectory(const float* signal, long long n_sig, const float* rirs, int n_points, int n_mics,
                               long long rir_len, float* out, const gpurir_opts* opts);

/* Number of samples ceil(T fs) under reading C9 (a product within 1e-6 of an integer from above
 * counts as that integer). */
long long gpurir_nsamples(double T, double fs);

/* ---- host helpers (pure, thread-safe) ---------------------------------------------- */

/* Eq. 7: Sabine T60 = 0.161 V / sum_i S_i (1 - beta_i^2); +inf if no wall absorbs. */
double gpurir_sabine_t60(const float room_sz[3], const float beta[6]);

/* A17 (reading C17): uniform alpha = 0.161 V / (T60 S), beta_i = sign * sqrt(1 - alpha).
 * sign < 0 (default in the paper's spirit) gives negative coefficients.  alpha > 1 returns
 * EINFEASIBLE unless clamp != 0, which returns beta = 0 (anechoic) and sets *clamped = 1. */
int gpurir_beta_sabine(const float room_sz[3], double T60, int sign, int clamp, float beta_out[6], int* clamped);

/* Non-uniform absorption (reading R9): alpha_i = weights[i] alpha0 with Sabine's Eq. 7
 * met exactly, alpha0 = 0.161 V / (T60 sum_i S_i weights[i]); beta_i = sign sqrt(1 - alpha_i).  weights
 * host float[6] >= 0, not all 0 (else EINVAL); some alpha_i > 1 returns EINFEASIBLE unless clamp != 0
 * (then beta = 0, *clamped = 1).  Equal weights give gpurir_beta_sabine's result. */
int gpurir_beta_sabine_weighted(const float room_sz[3], double T60, const float weights[6], int sign, int clamp,
                                float beta_out[6], int* clamped);

/* A18: time at which the exponential decay reaches att_dB: att_dB / 60 * T60. */
double gpurir_att2t_sabine(double att_dB, double T60);

/* A19 (reading C6): images per axis reaching time T without lost reflections,
 * N = 2 (ceil(c T / L) + 1) + 1 (odd). */
int gpurir_t2n(double T, const float room_sz[3], double c, int nb_img_out[3]);

/* ---- test / inspection hooks ---------------------------------------------------------------- */

/*
 * gpurir_image_params — the image-parameter stage (calcAmpTau; Eqs. 1-4 + A16) of
 * one (source, receiver) pair for every lattice image, in lattice order (n_x fastest, then n_y,
 * then n_z), computed by the same device code the accumulation kernel inlines.
 *   src, rcv, orv  host float[3] (orv ignored for omni)
 *   ors, spkr_pattern  source orientation host float[3] and pattern (f3; ors ignored / may be NULL for omni)
 *   x_out  device double[N]  delay in samples, tau_n * fs
 *   A_out  device float[N]   amplitude beta_n g_rcv g_src / (4 pi d_n)
 * Synchronises the stream.  Returns EDEGENERATE if some d_n = 0.
 */
int gpurir_image_params(const float room_sz[3], const float beta[6], const float src[3], const float rcv[3],
                        const float orv[3], int mic_pattern, const float ors[3], int spkr_pattern,
                        const int nb_img[3], double fs, double c, double* x_out, float* A_out, void* stream);

/* Windowed-sinc table of Eq. 9 (erratum C11) exactly as uploaded for GPURIR_LUT: entries
 * LUT[n], n = -half..half, written to host lut_out[0 .. 2 half] when lut_out != NULL and
 * cap >= 2 half + 1.  Returns half (>= 0) or -GPURIR_EINVAL. */
long long gpurir_lut_table(double Tw, double fs, int Q, float* lut_out, long long cap);

/* Polyphase expansion of Eq. 6 exactly as uploaded for GPURIR_POLY (reading R11): delta'(m - phi) ~=
 * sum_{d<8} P[m - mlo][d] T_d(2 phi - 1), phi in [0, 1), for taps m = mlo .. mlo + ntaps - 1 (the last
 * taps are zero padding to a multiple of 8).  Writes *mlo and, when P_out != NULL and cap >= 8 ntaps, the
 * host float[ntaps][8] table.  Returns ntaps, or -GPURIR_EINVAL (Tw fs > 1022 or not positive). */
int gpurir_poly_table(double Tw, double fs, int* mlo, float* P_out, long long cap);

/* The FIR form of that expansion exactly as GPURIR_POLY uploads it (reading R13): the channels
 * rotated per parity, G' = Q G (Q orthogonal, block diagonal over even / odd d, rows the eigenvectors of the
 * Gram matrix of the taps outside the window below), so that rotated channels 0..3 keep all ntaps taps and
 * channels 4..7 only the nn taps mi = nmi0 .. nmi0 + nn - 1 around m = 0, 1: delta'(m - phi) ~=
 * sum_r P'_r[m] (Q T(2 phi - 1))_r.  Writes *mlo, *nmi0, *nn and, when out != NULL and cap >= 4 ntaps + 4 nn + 32,
 * the host float table [far: 2 pairs][ntaps][2] (channels (0,1), (2,3)), [near: 2 pairs][nn][2] (channels (4,5),
 * (6,7)), Q [parity][k][i] (rotated channel 2k + parity = sum_i Q G_{2i + parity}).  Returns ntaps, or
 * -GPURIR_EINVAL. */
int gpurir_poly_fir_table(double Tw, double fs, int* mlo, int* nmi0, int* nn, float* out, long long cap);

/* Read and (if reset) clear the current device's status word (see file header). Synchronises. */
int gpurir_device_status(int reset);

const char* gpurir_strerror(int status);
/* Last CUDA error string recorded by this thread ("" if none). */
const char* gpurir_last_cuda_error(void);
/* Library version string. */
const char* gpurir_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GPURIR_H */

// Pipe-throughput microbenchmark for the B200 (sm_100a) roofline of the ISM
// accumulation kernel (SURVEY.md §7 hard part 9: "Measure FFMA, FFMA2,
// MUFU.RCP, DFMA and HFMA2 peaks with a microbenchmark on the box").
//
// Each kernel runs ILP independent dependency chains per thread for ITERS
// iterations; we report lane-operations per SM per clock, where the clock is
// measured with clock64() inside the kernel (so DVFS does not skew the ratio)
// and also ops/s from CUDA events.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 4096

__device__ unsigned long long g_cycles[4096];

#define TIMED_BEGIN                                   \
  unsigned long long t0 = clock64();
#define TIMED_END(sink)                               \
  unsigned long long t1 = clock64();                  \
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0; \
  if (sink == 12345.f) out[threadIdx.x] = sink;

__global__ void k_ffma(float* out, float a, float b) {
  float x[ILP];
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 0.001f + i;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = fmaf(x[i], a, b);
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  TIMED_END(s)
}

// 3 distinct register sources (the ISM Horner form: q = q*e + c with e varying)
__global__ void k_ffma_reg(float* out, float a, float b) {
  float x[ILP], y[ILP];
  for (int i = 0; i < ILP; i++) { x[i] = threadIdx.x * 0.001f + i; y[i] = a + i; }
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = fmaf(x[i], y[i], y[(i + 1) % ILP]);
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  TIMED_END(s)
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[ILP];
  float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int i = 0; i < ILP; i++) x[i] = make_float2(threadIdx.x * 0.001f + i, i);
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = __ffma2_rn(x[i], A, B);
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += x[i].x + x[i].y;
  TIMED_END(s)
}

__global__ void k_fmnmx(float* out, float a, float b) {
  float x[ILP];
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 0.001f + i;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = fmaxf(x[i], x[(i + 1) % ILP]) ;
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  TIMED_END(s)
}

__global__ void k_rcp(float* out, float a, float b) {
  float x[ILP];
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 0.001f + i + 1.f;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      float r;
      asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i]));
      x[i] = r;
    }
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  TIMED_END(s)
}

__global__ void k_ex2(float* out, float a, float b) {
  float x[ILP];
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 0.0001f + i * 0.01f;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      float r;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i]));
      x[i] = r;
    }
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  TIMED_END(s)
}

// mixed: 1 rcp per 10 ffma (the ISM tap mix)
__global__ void k_mix(float* out, float a, float b) {
  float x[ILP];
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 0.001f + i + 1.f;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) {
      float r;
      asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i]));
      float y = r;
#pragma unroll
      for (int j = 0; j < 10; j++) y = fmaf(y, a, b);
      x[i] = y;
    }
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  TIMED_END(s)
}

__global__ void k_dfma(float* out, float a, float b) {
  double x[ILP];
  double A = a, B = b;
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 0.001 + i;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = fma(x[i], A, B);
  }
  double s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  float fs = (float)s;
  TIMED_END(fs)
}

__global__ void k_hfma2(float* out, float a, float b) {
  __half2 x[ILP];
  __half2 A = __floats2half2_rn(a, a), B = __floats2half2_rn(b, b);
  for (int i = 0; i < ILP; i++) x[i] = __floats2half2_rn(threadIdx.x * 0.001f, i * 0.01f);
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = __hfma2(x[i], A, B);
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += __low2float(x[i]) + __high2float(x[i]);
  TIMED_END(s)
}

__global__ void k_imad(float* out, float a, float b) {
  unsigned x[ILP];
  unsigned A = (unsigned)a | 3u, B = (unsigned)b;
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x + i;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = x[i] * A + B;
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += (float)x[i];
  TIMED_END(s)
}

__global__ void k_lop3(float* out, float a, float b) {
  unsigned x[ILP];
  unsigned A = (unsigned)a | 3u, B = (unsigned)b;
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x + i;
  TIMED_BEGIN
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = (x[i] ^ A) & (x[(i + 1) % ILP] | B);
  }
  float s = 0; for (int i = 0; i < ILP; i++) s += (float)x[i];
  TIMED_END(s)
}

typedef void (*kfn)(float*, float, float);

static void run(const char* name, kfn k, double ops_per_iter_per_thread, int threads, int blocks_per_sm, int nsm) {
  float* out;
  cudaMalloc(&out, 4096 * sizeof(float));
  int blocks = nsm * blocks_per_sm;
  k<<<blocks, threads>>>(out, 1.0001f, 0.5f);  // warm
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, 1.0001f, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc[4096];
  cudaMemcpyFromSymbol(cyc, g_cycles, blocks * sizeof(unsigned long long));
  double maxc = 0; for (int i = 0; i < blocks; i++) if (cyc[i] > maxc) maxc = cyc[i];
  double total_ops = (double)blocks * threads * ITERS * ILP * ops_per_iter_per_thread;
  double per_sm_clk = total_ops / nsm / maxc;
  printf("%-10s %8.2f lane-ops/clk/SM  %9.3f Tops/s  (%.3f ms, clk est %.0f MHz) err=%s\n", name, per_sm_clk,
         total_ops / (ms * 1e-3) / 1e12, ms, maxc / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int nsm = p.multiProcessorCount;
  printf("device %s SMs %d clock %d kHz smemPerBlockOptin %zu\n", p.name, nsm, p.clockRate, p.sharedMemPerBlockOptin);
  for (int bps : {2, 4}) {
    printf("--- 256 threads x %d blocks/SM\n", bps);
    run("ffma", k_ffma, 1, 256, bps, nsm);
    run("ffma_reg", k_ffma_reg, 1, 256, bps, nsm);
    run("ffma2", k_ffma2, 2, 256, bps, nsm);
    run("fmnmx", k_fmnmx, 1, 256, bps, nsm);
    run("rcp", k_rcp, 1, 256, bps, nsm);
    run("ex2", k_ex2, 1, 256, bps, nsm);
    run("mix10:1", k_mix, 11, 256, bps, nsm);
    run("dfma", k_dfma, 1, 256, bps, nsm);
    run("hfma2", k_hfma2, 2, 256, bps, nsm);
    run("imad", k_imad, 1, 256, bps, nsm);
    run("lop3", k_lop3, 1, 256, bps, nsm);
  }
  return 0;
}

// tc_probe.cu — validates the tcgen05 building blocks the trajectory kernel uses (kind::tf32, cta_group::1,
// M = 128, N = 256, K-major operands in the no-swizzle canonical layout, D in TMEM, 32x32b loads): one CTA
// computes D = A B for small-integer A [128 x K] and B [K x 256] (exact in tf32 and fp32) and compares with
// the CPU.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tools/tc_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1810_11359_b200/csrc/tc_common.cuh"

using namespace gpurir::tc;

constexpr int M = 128, N = 256, K = 64;  // two 32-element chunks

__global__ void probe(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);                 // [K/32 chunks][128 rows x 32] canonical
  float* sB = sA + M * K;                                      // [K/32 chunks][256 cols x 32]
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int c = 0; c < K / 32; c++) {
    for (int i = tid; i < M * 32; i += blockDim.x) {
      const int r = i / 32, kk = i % 32;
      sA[c * M * 32 + canon_off(r, kk) / 4] = A[r * K + 32 * c + kk];
    }
    for (int i = tid; i < N * 32; i += blockDim.x) {
      const int n = i / 32, kk = i % 32;
      sB[c * N * 32 + canon_off(n, kk) / 4] = B[(32 * c + kk) * N + n];
    }
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  if (tid == 0) mbar_init(&bar, 1);
  fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    for (int c = 0; c < K / 32; c++)
      for (int k = 0; k < 4; k++) {
        const uint64_t da = smem_desc(sA + c * M * 32 + k * 64);  // +2 core matrices (256 B) per K step of 8
        const uint64_t db = smem_desc(sB + c * N * 32 + k * 64);
        mma_tf32(tmem, da, db, idesc, (c | k) != 0);
      }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      const int row = 32 * warp + (tid & 31);
      for (int j = 0; j < 16; j++) D[row * N + c0 + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int rate_main();
int sw_main();
int pair_main();
int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'p') return pair_main();
  if (argc > 1 && argv[1][0] == 'r') return rate_main();
  if (argc > 1 && argv[1][0] == 's') return sw_main();
  std::vector<float> A(M * K), B(K * N), D(M * N), R(M * N, 0.f);
  srand(1);
  for (auto& x : A) x = (float)(rand() % 17 - 8);
  for (auto& x : B) x = (float)(rand() % 17 - 8);
  for (int i = 0; i < M; i++)
    for (int n = 0; n < N; n++) {
      double s = 0;
      for (int k = 0; k < K; k++) s += (double)A[i * K + k] * B[k * N + n];
      R[i * N + n] = (float)s;
    }
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  const size_t sm = (size_t)(M + N) * K * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  probe<<<1, 256, sm>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M * N; i++)
    if (D[i] != R[i]) {
      if (bad < 8) printf("mismatch row %d col %d: got %g want %g\n", i / N, i % N, D[i], R[i]);
      bad++;
    }
  printf("tc_probe: %d mismatches of %d\n", bad, M * N);
  return bad != 0;
}

// ---- MMA throughput of one CTA: the trajectory kernel's chunk (3 x 4 MMAs of M128 N256 K8, tf32) repeated ----
__global__ void probe_rate(int reps, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (96 * 1024) / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1.0f / (1 + (i & 7));
  fence_proxy_async();
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  if (tid == 0) mbar_init(&bar, 1);
  fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, 256);
    const unsigned char *Ah = smem, *Al = smem + 16384, *Bh = smem + 32768, *Bl = smem + 65536;
    const long long t0 = clock64();
    for (int q = 0; q < reps; q++)
      for (int k = 0; k < 4; k++) {
        const uint64_t dah = smem_desc(Ah + 256 * k), dal = smem_desc(Al + 256 * k);
        const uint64_t dbh = smem_desc(Bh + 256 * k), dbl = smem_desc(Bl + 256 * k);
        mma_tf32(tmem, dah, dbh, idesc, q > 0 || k > 0);
        mma_tf32(tmem, dah, dbl, idesc, true);
        mma_tf32(tmem, dal, dbh, idesc, true);
      }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    cycles[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int rate_main() {
  long long* dc;
  cudaMalloc(&dc, 8);
  cudaFuncSetAttribute(probe_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int reps : {10, 100, 1000}) {
    probe_rate<<<1, 128, 96 * 1024>>>(reps, dc);
    long long c = 0;
    cudaDeviceSynchronize();
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    const double macs = (double)reps * 12 * 128 * 256 * 8;
    printf("rate: %d chunks  %lld cycles  %.1f cycles/MMA  %.0f MAC/clk (tf32)\n", reps, c, (double)c / (12.0 * reps),
           macs / c);
  }
  return 0;
}

// ---- SWIZZLE_128B K-major operands ([rows x 32 fp32]: 8-row atoms of 1024 B, 16-B chunk j of row r at j ^ r),
// K advanced by +32 B per step; and the tf32 conversion of fp32 operands (truncation or rounding) ----
__host__ __device__ inline int sw_off(int row, int kk) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((((kk >> 2) ^ (row & 7)) & 7) << 4) + (kk & 3) * 4;
}
__global__ void probe_sw(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = sA + M * 32;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * 32; i += blockDim.x) sA[sw_off(i / 32, i % 32) / 4] = A[(i / 32) * K + i % 32];
  for (int i = tid; i < N * 32; i += blockDim.x) sB[sw_off(i / 32, i % 32) / 4] = B[(i % 32) * N + i / 32];
  fence_proxy_async();
  if (warp == 0) tmem_alloc(&tmem_base, 256);
  if (tid == 0) mbar_init(&bar, 1);
  fence_mbar_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N);
    for (int k = 0; k < 4; k++) mma_tf32(tmem, smem_desc_sw128(sA) + (uint64_t)(2 * k), smem_desc_sw128(sB) + (uint64_t)(2 * k), idesc, k != 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4)
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      for (int j = 0; j < 16; j++) D[(32 * warp + (tid & 31)) * N + c0 + j] = v[j];
    }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int sw_main() {
  std::vector<float> A(M * K), B(K * N), D(M * N);
  srand(2);
  for (auto& x : A) x = (float)(rand() % 17 - 8);
  for (auto& x : B) x = (float)(rand() % 17 - 8);
  // column 0 of B: 1 + 2^-12 + 2^-20 (low mantissa bits below tf32), row 0 of A: 1 at k = 0, 0 elsewhere
  for (int k = 0; k < K; k++) A[k] = k == 0 ? 1.f : 0.f;
  B[0] = 1.0f + 0.00048828125f + 0.00000095367431640625f;  // 1 + 2^-11 + 2^-20
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe_sw, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe_sw<<<1, 256, 64 * 1024>>>(dA, dB, dD);
  printf("sw kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 1; i < M; i++)  // rows 1.. (row 0 is the conversion probe)
    for (int n = 1; n < N; n++) {  // column 0 holds the conversion probe
      double s = 0;
      for (int k = 0; k < 32; k++) s += (double)A[i * K + k] * B[k * N + n];
      if (D[i * N + n] != (float)s) { if (bad < 5) printf("sw mismatch %d %d: %g vs %g\n", i, n, D[i * N + n], s); bad++; }
    }
  printf("sw128: %d mismatches; tf32(1 + 2^-11 + 2^-20) = %.10f (truncation: 1, round to nearest: 1.0009765625)\n",
         bad, D[0]);
  return bad != 0;
}

// ---- CTA pair: cluster of 2, M = 256 (128 rows per CTA), N = 256 (128 columns of B per CTA), K = 32, SW128 ----
__global__ void __cluster_dims__(2, 1, 1) probe_pair(const float* A, const float* B, float* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* sA = reinterpret_cast<float*>(smem);            // this CTA's 128 rows x 32
  float* sB = sA + 128 * 32;                              // this CTA's 128 columns x 32
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < 128 * 32; i += blockDim.x) {
    sA[sw_off(i / 32, i % 32) / 4] = A[(128 * rank + i / 32) * 32 + i % 32];
    sB[sw_off(i / 32, i % 32) / 4] = B[(i % 32) * 256 + 128 * rank + i / 32];
  }
  fence_proxy_async();
  if (warp == 0) tmem_alloc_pair(&tmem_base, 256);
  if (tid == 0) mbar_init(&bar, 1);
  fence_mbar_init();
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = idesc_tf32(256, 256);
    for (int k = 0; k < 4; k++)
      mma_tf32_pair(tmem, smem_desc_sw128(sA) + 2 * k, smem_desc_sw128(sB) + 2 * k, idesc, k != 0);
    mma_commit_pair(&bar, 3);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4)
    for (int c0 = 0; c0 < 256; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * warp) << 16) + c0, v);
      for (int j = 0; j < 16; j++) D[(128 * rank + 32 * warp + (tid & 31)) * 256 + c0 + j] = v[j];
    }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) tmem_dealloc_pair(tmem, 256);
}

int pair_main() {
  std::vector<float> A(256 * 32), B(32 * 256), D(256 * 256);
  srand(3);
  for (auto& x : A) x = (float)(rand() % 17 - 8);
  for (auto& x : B) x = (float)(rand() % 17 - 8);
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  cudaFuncSetAttribute(probe_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe_pair<<<2, 128, 64 * 1024>>>(dA, dB, dD);
  printf("pair kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 256; i++)
    for (int n = 0; n < 256; n++) {
      double s = 0;
      for (int k = 0; k < 32; k++) s += (double)A[i * 32 + k] * B[k * 256 + n];
      if (D[i * 256 + n] != (float)s) { if (bad < 5) printf("pair mismatch %d %d: %g vs %g\n", i, n, D[i * 256 + n], s); bad++; }
    }
  printf("pair: %d mismatches of %d\n", bad, 256 * 256);
  return bad != 0;
}

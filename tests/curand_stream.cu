// curand_stream.cu — cuRAND's device-API Philox4_32_10 stream, for the RNG pin of tests/test_gpu_parity.py
// (test infrastructure; shares nothing with the library or the oracle).  SURVEY §8(c) RNG row / reading C16:
// the diffuse tail's noise word k of RIR r must equal the k-th curand() after curand_init(seed, r, 0).
#include <curand_kernel.h>
#include <stdint.h>

__global__ void curand_words_kernel(unsigned long long seed, unsigned long long r, unsigned long long k0, int n,
                                    uint32_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  curandStatePhilox4_32_10_t st;
  curand_init(seed, r, k0, &st);  // subsequence = the RIR, offset = the first sample
  for (int i = 0; i < n; i++) out[i] = curand(&st);
}

extern "C" int curand_words(unsigned long long seed, unsigned long long r, unsigned long long k0, int n,
                            uint32_t* out_dev) {
  curand_words_kernel<<<1, 32>>>(seed, r, k0, n, out_dev);
  return (int)cudaDeviceSynchronize();
}

// Graph-replay granularity probe (diagnostic): a kernel that spins `cycles` SM clocks in every CTA, launched with
// or without a thread-block cluster attribute; tools/replay_quantum.py replays it from a CUDA graph.
#include <cuda_runtime.h>
__global__ void spin_kernel(long long cycles, int* sink) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && cycles < 0) *sink = 1;
}
extern "C" int spin_launch(long long cycles, int blocks, int threads, int cluster, void* stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks, 1, 1);
  cfg.blockDim = dim3((unsigned)threads, 1, 1);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)(cluster > 0 ? cluster : 1);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cluster > 0 ? 1 : 0;
  return (int)cudaLaunchKernelEx(&cfg, spin_kernel, cycles, (int*)nullptr);
}

// Does compute-sanitizer initcheck track device memory written by
// cudaMemcpyBatchAsync? Copies two pinned host buffers with one batch call,
// then a kernel reads them (a clean run prints "ok" with 0 initcheck errors).
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_sum(const int* a, int n, int* out) {
  int s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += a[i];
  atomicAdd(out, s);
}
int main() {
  const int n = 4096;
  int *h0, *h1, *d, *out;
  cudaHostAlloc(&h0, n * 4, cudaHostAllocPortable);
  cudaHostAlloc(&h1, n * 4, cudaHostAllocPortable);
  for (int i = 0; i < n; ++i) h0[i] = h1[i] = 1;
  cudaMalloc(&d, 2 * n * 4);
  cudaMalloc(&out, 4);
  cudaMemset(out, 0, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  void* dsts[2] = {d, d + n};
  void* srcs[2] = {h0, h1};
  size_t sizes[2] = {n * 4, n * 4};
  cudaMemcpyAttributes attr{};
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  attr.srcLocHint.type = cudaMemLocationTypeHost;
  attr.dstLocHint.type = cudaMemLocationTypeDevice;
  size_t idx = 0, fail = 0;
  cudaError_t e = cudaMemcpyBatchAsync(dsts, srcs, sizes, 2, &attr, &idx, 1, &fail, s);
  k_sum<<<1, 256, 0, s>>>(d, 2 * n, out);
  int r = 0;
  cudaMemcpyAsync(&r, out, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  printf("batch copy %s, sum %d (want %d) -> %s\n", cudaGetErrorString(e), r, 2 * n, r == 2 * n ? "ok" : "BAD");
  return r == 2 * n ? 0 : 1;
}

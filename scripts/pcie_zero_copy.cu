// Probe (tools only): H2D rate of SM loads from mapped pinned host memory, alone and next to a
// copy-engine transfer on another stream.  Does the link carry more than the DMA engine alone?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o scripts/_zc.so scripts/pcie_zero_copy.cu
#include <cuda_runtime.h>
#include <cstdint>

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  // 4 independent 16-byte loads in flight per thread
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a; dst[i + stride] = b; dst[i + 2 * stride] = c; dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

extern "C" {

// returns {zc_alone, dma_alone, zc_with_dma, dma_with_zc, combined} in GB/s
int zc_probe(size_t bytes, int blocks, int threads, double* out) {
  void *h0, *h1, *d0, *d1;
  if (cudaHostAlloc(&h0, bytes, cudaHostAllocMapped) != cudaSuccess) return 1;
  if (cudaHostAlloc(&h1, bytes, cudaHostAllocDefault) != cudaSuccess) return 2;
  if (cudaMalloc(&d0, bytes) != cudaSuccess || cudaMalloc(&d1, bytes) != cudaSuccess) return 3;
  for (size_t i = 0; i < bytes; i += 4096) { ((char*)h0)[i] = 1; ((char*)h1)[i] = 1; }
  void* hd0;
  cudaHostGetDevicePointer(&hd0, h0, 0);
  cudaStream_t s0, s1;
  cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaEvent_t a0, b0, a1, b1;
  cudaEventCreate(&a0); cudaEventCreate(&b0); cudaEventCreate(&a1); cudaEventCreate(&b1);
  const size_t n16 = bytes / 16;
  double best[5] = {0, 0, 0, 0, 0};
  for (int rep = 0; rep < 4; ++rep) {
    float ms;
    cudaEventRecord(a0, s0);
    zc_read<<<blocks, threads, 0, s0>>>((const uint4*)hd0, (uint4*)d0, n16);
    cudaEventRecord(b0, s0);
    cudaStreamSynchronize(s0);
    cudaEventElapsedTime(&ms, a0, b0);
    if (bytes / (ms * 1e6) > best[0]) best[0] = bytes / (ms * 1e6);
    cudaEventRecord(a1, s1);
    cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
    cudaEventRecord(b1, s1);
    cudaStreamSynchronize(s1);
    cudaEventElapsedTime(&ms, a1, b1);
    if (bytes / (ms * 1e6) > best[1]) best[1] = bytes / (ms * 1e6);
    // both at once
    cudaDeviceSynchronize();
    cudaEventRecord(a0, s0);
    cudaStreamWaitEvent(s1, a0, 0);
    cudaEventRecord(a1, s1);
    zc_read<<<blocks, threads, 0, s0>>>((const uint4*)hd0, (uint4*)d0, n16);
    cudaMemcpyAsync(d1, h1, bytes, cudaMemcpyHostToDevice, s1);
    cudaEventRecord(b0, s0);
    cudaEventRecord(b1, s1);
    cudaDeviceSynchronize();
    float m0, m1, mall;
    cudaEventElapsedTime(&m0, a0, b0);
    cudaEventElapsedTime(&m1, a1, b1);
    cudaEventElapsedTime(&mall, a0, m0 > m1 ? b0 : b1);
    if (bytes / (m0 * 1e6) > best[2]) best[2] = bytes / (m0 * 1e6);
    if (bytes / (m1 * 1e6) > best[3]) best[3] = bytes / (m1 * 1e6);
    if (2.0 * bytes / (mall * 1e6) > best[4]) best[4] = 2.0 * bytes / (mall * 1e6);
  }
  for (int i = 0; i < 5; ++i) out[i] = best[i];
  cudaFreeHost(h0); cudaFreeHost(h1); cudaFree(d0); cudaFree(d1);
  return cudaGetLastError() == cudaSuccess ? 0 : 4;
}
}

// Probe (tools only): where the event-timed duration of a streaming kernel goes when its launch
// waits on a saturated H2D copy stream, as in the decode step (K2 after the on-demand copy).
//
// A 148 x 512 kernel streams `bytes` of device memory (16-byte loads) and stamps %globaltimer at
// its first CTA start / last CTA end.  The copy stream moves 32 MB H2D chunks back to back; the
// compute stream waits for the k-th chunk, then [timing event a] kernel [timing event b].
// Reported per variant: mean event interval, mean in-kernel span, their difference.
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/event_probe scripts/event_probe.cu -lcuda
//   /tmp/event_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

template <int PAD>
struct Params {
  const uint4* src;
  size_t n16;
  unsigned long long* ts;   // [0] = min start, [1] = max end
  float* sink;
  int pad[PAD];
};

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int PAD>
__global__ void __launch_bounds__(512, 1) stream_k(const __grid_constant__ Params<PAD> p) {
  if (threadIdx.x == 0) atomicMin(p.ts, gt());
  const size_t per = (p.n16 + gridDim.x - 1) / gridDim.x;
  const size_t b = per * blockIdx.x, e = b + per < p.n16 ? b + per : p.n16;
  uint32_t acc = 0;
  for (size_t i = b + threadIdx.x; i < e; i += blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * blockDim.x < e) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                                                : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w)
                                                : "l"(p.src + i + k * blockDim.x));
      else v[k] = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc ^= v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678u) p.sink[0] = 1.f;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(p.ts + 1, gt());
}

struct Res { double ev_us, k_us; };

template <int PAD>
static int run(const char* name, bool load, int waitmode, size_t bytes, const uint4* src, float* sink,
               unsigned long long* ts_d, uint8_t* hsrc, uint8_t* ddst, cudaStream_t cs, cudaStream_t ks,
               uint32_t* flag_d) {
  const int iters = 40;
  const size_t chunk = 32ull << 20;
  std::vector<cudaEvent_t> ea(iters), eb(iters), ec(iters);
  for (int i = 0; i < iters; ++i) {
    CK(cudaEventCreate(&ea[i]));
    CK(cudaEventCreate(&eb[i]));
    CK(cudaEventCreateWithFlags(&ec[i], cudaEventDisableTiming));
  }
  std::vector<unsigned long long> init(2 * iters);
  for (int i = 0; i < iters; ++i) { init[2 * i] = ~0ull; init[2 * i + 1] = 0; }
  CK(cudaMemcpy(ts_d, init.data(), 16 * iters, cudaMemcpyHostToDevice));
  CK(cudaMemset(flag_d, 0, 4));
  CK(cudaDeviceSynchronize());
  Params<PAD> p{};
  p.src = src;
  p.n16 = bytes / 16;
  p.sink = sink;
  for (int i = 0; i < iters; ++i) {
    if (load) {   // keep the link busy: 4 chunks ahead of each kernel
      for (int k = 0; k < 4; ++k)
        CK(cudaMemcpyAsync(ddst + (size_t)((i * 4 + k) % 16) * chunk, hsrc + (size_t)((i * 4 + k) % 16) * chunk, chunk,
                           cudaMemcpyHostToDevice, cs));
      if (waitmode == 1) {
        CK(cudaEventRecord(ec[i], cs));
        CK(cudaStreamWaitEvent(ks, ec[i], 0));
      } else if (waitmode == 2) {
        if (cuStreamWriteValue32((CUstream)cs, (CUdeviceptr)flag_d, (cuuint32_t)(i + 1), 0) != CUDA_SUCCESS) return 2;
        if (cuStreamWaitValue32((CUstream)ks, (CUdeviceptr)flag_d, (cuuint32_t)(i + 1), CU_STREAM_WAIT_VALUE_GEQ) !=
            CUDA_SUCCESS) return 3;
      }
    }
    p.ts = ts_d + 2 * i;
    CK(cudaEventRecord(ea[i], ks));
    stream_k<PAD><<<148, 512, 0, ks>>>(p);
    CK(cudaGetLastError());
    CK(cudaEventRecord(eb[i], ks));
  }
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> ts(2 * iters);
  CK(cudaMemcpy(ts.data(), ts_d, 16 * iters, cudaMemcpyDeviceToHost));
  double ev = 0, kk = 0;
  int n = 0;
  for (int i = 4; i < iters; ++i) {
    float ms;
    CK(cudaEventElapsedTime(&ms, ea[i], eb[i]));
    ev += ms * 1e3;
    kk += (ts[2 * i + 1] - ts[2 * i]) * 1e-3;
    ++n;
  }
  printf("{\"variant\": \"%s\", \"pad_bytes\": %d, \"MB\": %.1f, \"event_us\": %.2f, \"kernel_us\": %.2f, "
         "\"overhead_us\": %.2f}\n", name, PAD * 4, bytes / 1e6, ev / n, kk / n, (ev - kk) / n);
  for (int i = 0; i < iters; ++i) {
    cudaEventDestroy(ea[i]);
    cudaEventDestroy(eb[i]);
    cudaEventDestroy(ec[i]);
  }
  return 0;
}

int main() {
  const size_t big = 1ull << 30;
  uint4* src;
  float* sink;
  unsigned long long* ts;
  uint8_t *hsrc, *ddst;
  uint32_t* flag;
  CK(cudaMalloc(&src, big));
  CK(cudaMemset(src, 1, big));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&ts, 16 * 64));
  CK(cudaMalloc(&flag, 64));
  CK(cudaMallocHost(&hsrc, 16 * (32ull << 20)));
  CK(cudaMalloc(&ddst, 16 * (32ull << 20)));
  cudaStream_t cs, ks;
  CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
  int lo_pri = 0, hi_pri = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
  cudaStream_t ks_hi;
  CK(cudaStreamCreateWithPriority(&ks_hi, cudaStreamNonBlocking, hi_pri));
  for (size_t mb : {370ull, 64ull}) {
    const size_t bytes = mb << 20;
    if (run<4>("load_waitevent_hiprio", true, 1, bytes, src, sink, ts, hsrc, ddst, cs, ks_hi, flag)) return 1;
    if (run<4>("load_waitvalue_hiprio", true, 2, bytes, src, sink, ts, hsrc, ddst, cs, ks_hi, flag)) return 1;
    if (run<4>("idle_nowait", false, 0, bytes, src, sink, ts, hsrc, ddst, cs, ks, flag)) return 1;
    if (run<4>("load_nowait", true, 0, bytes, src, sink, ts, hsrc, ddst, cs, ks, flag)) return 1;
    if (run<4>("load_waitevent", true, 1, bytes, src, sink, ts, hsrc, ddst, cs, ks, flag)) return 1;
    if (run<1024>("load_waitevent", true, 1, bytes, src, sink, ts, hsrc, ddst, cs, ks, flag)) return 1;
    if (run<4>("load_waitvalue", true, 2, bytes, src, sink, ts, hsrc, ddst, cs, ks, flag)) return 1;
  }
  return 0;
}

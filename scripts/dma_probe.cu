// Probe (tools only): fixed cost of an H2D copy on the DMA engine, as the decode step issues them
// (one cudaMemcpyAsync per segment, 2-10 MB segments on Qwen3 / DeepSeek shapes).
//   single   one copy of S bytes after an idle link (event-timed): intercept = start-up cost
//   chain    n copies of S back to back on one stream: per-copy cost above bytes / rate
//   two      the same n copies alternating over two streams
//
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/dma_probe scripts/dma_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

// holds the stream while the host enqueues the copies (host enqueue speed out of the timing)
__global__ void hold(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { __nanosleep(1000); asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
}

int main() {
  const size_t hbytes = 2ull << 30;
  uint8_t *h, *d;
  CK(cudaMallocHost(&h, hbytes));
  CK(cudaMalloc(&d, hbytes));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t a, b, j;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
  // steady-state rate: 1 GiB in one copy
  float ms;
  for (int w = 0; w < 2; ++w) {
    CK(cudaEventRecord(a, s0));
    CK(cudaMemcpyAsync(d, h, 1ull << 30, cudaMemcpyHostToDevice, s0));
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
  }
  CK(cudaEventElapsedTime(&ms, a, b));
  const double rate = (1ull << 30) / (ms * 1e-3) / 1e9;   // GB/s
  printf("{\"probe\": \"rate_1GiB\", \"GBps\": %.2f}\n", rate);
  for (size_t mb : {1ull, 2ull, 4ull, 8ull, 16ull, 64ull}) {
    const size_t S = mb << 20;
    double best = 1e30, sum = 0;
    for (int r = 0; r < 10; ++r) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s0));
      CK(cudaMemcpyAsync(d + (r % 4) * S, h + (r % 4) * S, S, cudaMemcpyHostToDevice, s0));
      CK(cudaEventRecord(b, s0));
      CK(cudaEventSynchronize(b));
      CK(cudaEventElapsedTime(&ms, a, b));
      best = ms < best ? ms : best;
      sum += ms;
    }
    printf("{\"probe\": \"single\", \"MB\": %zu, \"best_us\": %.2f, \"mean_us\": %.2f, \"over_rate_us\": %.2f}\n", mb,
           best * 1e3, sum * 1e2, best * 1e3 - S / (rate * 1e3));
  }
  for (size_t kb : {512ull, 1024ull, 2048ull, 4096ull, 8192ull}) {
    const size_t S = kb << 10;
    const int n = (int)std::min<size_t>(64, hbytes / S);
    std::vector<void*> dst(n), src(n);
    std::vector<size_t> sz(n, S);
    for (int i = 0; i < n; ++i) {   // scattered sources, like segments of different experts
      src[i] = h + (size_t)((i * 7) % n) * S;
      dst[i] = d + (size_t)i * S;
    }
    for (int mode = 0; mode < 2; ++mode) {
      double best = 1e30;
      for (int r = 0; r < 5; ++r) {
        CK(cudaDeviceSynchronize());
        hold<<<1, 1, 0, s0>>>(3000000ull);
        CK(cudaEventRecord(a, s0));
        if (mode == 0) {
          for (int i = 0; i < n; ++i) CK(cudaMemcpyAsync(dst[i], src[i], S, cudaMemcpyHostToDevice, s0));
        } else if (mode == 1) {
          CK(cudaStreamWaitEvent(s1, a, 0));
          for (int i = 0; i < n; ++i) CK(cudaMemcpyAsync(dst[i], src[i], S, cudaMemcpyHostToDevice, (i & 1) ? s1 : s0));
          CK(cudaEventRecord(j, s1));
          CK(cudaStreamWaitEvent(s0, j, 0));
        }
        CK(cudaEventRecord(b, s0));
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
      }
      const double ideal = (double)n * S / (rate * 1e3);
      printf("{\"probe\": \"%s\", \"KB\": %zu, \"n\": %d, \"us\": %.1f, \"GBps\": %.2f, \"per_copy_over_us\": %.2f}\n",
             mode == 0 ? "chain" : "two_streams", kb, n, best * 1e3,
             (double)n * S / (best * 1e-3) / 1e9, (best * 1e3 - ideal) / n);
    }
  }
  return 0;
}

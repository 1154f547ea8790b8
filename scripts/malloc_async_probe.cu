// Probe: device-time cost of a stream-ordered cudaMallocAsync / cudaFreeAsync
// cycle of plan-sized blocks (tree arena ~50 MB, level buffers ~360 MB), as
// sft_plan / sft_destroy do per step.  Prints device microseconds between
// %globaltimer stamps around each call (stamps in device memory: a managed
// page would fault on the first GPU write of every iteration).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void stamp(unsigned long long* o) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); *o = t; }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaMemPool_t pool; cudaDeviceGetDefaultMemPool(&pool, 0);
  unsigned long long thr = ~0ull; cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  unsigned long long* ts; cudaMallocHost(&ts, 64 * sizeof(unsigned long long)); unsigned long long* dts; cudaMalloc(&dts, 64 * sizeof(unsigned long long));
  for (int it = 0; it < 6; ++it) {
    void *a = nullptr, *b = nullptr;
    stamp<<<1, 1, 0, s>>>(dts + 0);
    cudaMallocAsync(&a, 50u << 20, s);
    stamp<<<1, 1, 0, s>>>(dts + 1);
    cudaMemsetAsync(a, 0, 8u << 20, s);
    stamp<<<1, 1, 0, s>>>(dts + 2);
    cudaMallocAsync(&b, 360u << 20, s);
    stamp<<<1, 1, 0, s>>>(dts + 3);
    cudaFreeAsync(b, s);
    cudaFreeAsync(a, s);
    stamp<<<1, 1, 0, s>>>(dts + 4);
    stamp<<<1, 1, 0, s>>>(dts + 5);
    cudaMemcpyAsync(ts, dts, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    printf("iter %d: malloc50 %.1f us, memset8 %.1f us, malloc360 %.1f us, free %.1f us, empty %.1f us\n", it,
           (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3, (ts[4] - ts[3]) * 1e-3,
           (ts[5] - ts[4]) * 1e-3);
  }
  return 0;
}

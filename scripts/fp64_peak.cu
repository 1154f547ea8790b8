// fp64_peak.cu -- FP64 throughput microbenchmark on B200.
// Measures DFMA (register operands; constant-bank operand) and DMMA
// (mma.sync.m8n8k4.f64) throughput, reports TFLOP/s and the SM clock seen.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double c_k[16];

template <int CH>
__global__ void dfma_reg(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void dfma_const(double* out, int iters) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], c_k[c & 15], c_k[(c + 1) & 15]);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

// my kernel's shape: acc += c_const * x_reg, 4 accumulators per (m) row, 9 x regs
template <int P>
__global__ void dfma_one_const(double* out, int iters) {
  double x[P];
#pragma unroll
  for (int l = 0; l < P; ++l) x[l] = threadIdx.x * 1e-3 + l;
  double s = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int m = 0; m < P; ++m) {
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        a0 = fma(c_k[(m + l) & 15], x[l], a0);
        a1 = fma(c_k[(m + l) & 15], x[(l + 1) % P], a1);
        a2 = fma(c_k[(m + l + 1) & 15], x[l], a2);
        a3 = fma(c_k[(m + l + 1) & 15], x[(l + 1) % P], a3);
      }
      x[m] += 1e-9 * (a0 + a1 + a2 + a3);
    }
  }
#pragma unroll
  for (int l = 0; l < P; ++l) s += x[l];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[2] = {0, 0}, c1[2] = {0, 0}, c2[2] = {0, 0}, c3[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c1[0]), "+d"(c1[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c2[0]), "+d"(c2[1]) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c3[0]), "+d"(c3[1]) : "d"(a), "d"(b));
  }
  double s = c0[0] + c0[1] + c1[0] + c1[1] + c2[0] + c2[1] + c3[0] + c3[1];
  if (s == 12345.678) out[0] = s;
}


// latency of one dependent DMMA (single warp, one accumulator chain)
__global__ void dmma_lat(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0[2] = {0, 0};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0[0]), "+d"(c0[1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (c0[0] + c0[1] == 12345.678) out[0] = c0[0];
}

// DMMA with CH independent chains per warp
template <int CH>
__global__ void dmma_ch(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[CH][2];
#pragma unroll
  for (int j = 0; j < CH; ++j) c[j][0] = c[j][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

// DMMA (4 chains) and DFMA (8 chains) interleaved in the same warp: do the
// two pipes add up?
__global__ void mixed(double* out, int iters, double fa, double fb) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = fma(acc[j], fa, fb);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void clk(long long* o) {
  long long t0 = clock64();
  long long g0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
  while (clock64() - t0 < 200000000LL) {
  }
  long long g1;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
  o[0] = g1 - g0;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  double h[16];
  for (int i = 0; i < 16; ++i) h[i] = 0.999 + 1e-4 * i;
  cudaMemcpyToSymbol(c_k, h, sizeof(h));
  double* out;
  cudaMalloc(&out, 64);
  long long* ck;
  cudaMalloc(&ck, 8);
  const int iters = 20000, threads = 256, blocks = nsm * 8;
  {
    float ms = timeit([&] { dfma_reg<8><<<blocks, threads>>>(out, iters, 0.999, 1e-6); });
    double fl = 2.0 * 8 * iters * (double)threads * blocks;
    printf("{\"test\": \"dfma_reg_8chains\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, fl / ms / 1e9);
  }
  {
    float ms = timeit([&] { dfma_reg<4><<<blocks, threads>>>(out, iters * 2, 0.999, 1e-6); });
    double fl = 2.0 * 4 * iters * 2 * (double)threads * blocks;
    printf("{\"test\": \"dfma_reg_4chains\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, fl / ms / 1e9);
  }
  {
    float ms = timeit([&] { dfma_const<8><<<blocks, threads>>>(out, iters); });
    double fl = 2.0 * 8 * iters * (double)threads * blocks;
    printf("{\"test\": \"dfma_constbank_8chains\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, fl / ms / 1e9);
  }
  {
    const int it2 = iters / 40;
    float ms = timeit([&] { dfma_one_const<9><<<blocks, threads>>>(out, it2); });
    double fl = 2.0 * 4 * 81 * it2 * (double)threads * blocks;
    printf("{\"test\": \"dfma_one_const_rows_p9\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, fl / ms / 1e9);
  }
  for (int wps : {2, 4, 8, 12, 16, 24, 32}) {  // warps per SM, one CTA per SM
    const int it2 = iters / 40;
    float ms = timeit([&] { dfma_one_const<9><<<nsm, 32 * wps>>>(out, it2); });
    double fl = 2.0 * 4 * 81 * it2 * (double)(32 * wps) * nsm;
    printf("{\"test\": \"dfma_one_const_rows_p9\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", wps, fl / ms / 1e9);
  }
  {
    float ms = timeit([&] { dmma<<<blocks, threads>>>(out, iters / 4); });
    double fl = 2.0 * 8 * 8 * 4 * 4 * (iters / 4) * (double)(threads / 32) * blocks;
    printf("{\"test\": \"dmma_m8n8k4\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, fl / ms / 1e9);
  }
  {
    dmma_lat<<<1, 32>>>(out, ck, 10000);
    cudaDeviceSynchronize();
    long long cyc;
    cudaMemcpy(&cyc, ck, 8, cudaMemcpyDeviceToHost);
    printf("{\"test\": \"dmma_dependent_latency\", \"cycles\": %.1f}\n", cyc / 10000.0);
  }
  for (int wps : {4, 8, 16, 32}) {
    float ms = timeit([&] { dmma_ch<4><<<nsm, 32 * wps>>>(out, iters / 4); });
    double fl = 2.0 * 256 * 4 * (iters / 4) * (double)wps * nsm;
    printf("{\"test\": \"dmma_4chains\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", wps, fl / ms / 1e9);
  }
  for (int wps : {4, 8, 16}) {
    float ms = timeit([&] { dmma_ch<8><<<nsm, 32 * wps>>>(out, iters / 8); });
    double fl = 2.0 * 256 * 8 * (iters / 8) * (double)wps * nsm;
    printf("{\"test\": \"dmma_8chains\", \"warps_per_sm\": %d, \"tflops\": %.2f}\n", wps, fl / ms / 1e9);
  }
  {
    const int it2 = iters / 4;
    float ms = timeit([&] { mixed<<<blocks, threads>>>(out, it2, 0.999, 1e-6); });
    double fl_mma = 2.0 * 256 * 4 * it2 * (double)(threads / 32) * blocks;
    double fl_fma = 2.0 * 32 * 32 * it2 * (double)(threads / 32) * blocks;
    printf("{\"test\": \"mixed_dmma_dfma\", \"ms\": %.3f, \"tflops_total\": %.2f, \"tflops_dmma\": %.2f, \"tflops_dfma\": %.2f}\n",
           ms, (fl_mma + fl_fma) / ms / 1e9, fl_mma / ms / 1e9, fl_fma / ms / 1e9);
  }
  {
    clk<<<1, 1>>>(ck);
    long long ns;
    cudaMemcpy(&ns, ck, 8, cudaMemcpyDeviceToHost);
    printf("{\"test\": \"sm_clock\", \"mhz\": %.1f}\n", 200000000.0 / ns * 1e3);
  }
  printf("{\"sms\": %d}\n", nsm);
  return 0;
}

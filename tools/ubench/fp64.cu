// fp64 pipe microbenchmark: DFMA throughput vs ILP, DMMA (mma.sync m8n8k4 f64) throughput.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0001;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main1() {
  double* out; cudaMalloc(&out, 1 << 20);
  int sms = 148, iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    int threads = warps * 32;
    float ms1 = timeit([&] { dfma_kernel<1><<<sms, threads>>>(out, iters, 1.0000001, 1e-9); });
    float ms4 = timeit([&] { dfma_kernel<4><<<sms, threads>>>(out, iters, 1.0000001, 1e-9); });
    float ms8 = timeit([&] { dfma_kernel<8><<<sms, threads>>>(out, iters, 1.0000001, 1e-9); });
    double f = 2.0 * sms * threads * iters * 16;
    printf("DFMA warps/SM=%2d  ILP1 %.2f TF  ILP4 %.2f TF  ILP8 %.2f TF\n", warps, f * 1 / ms1 / 1e9,
           f * 4 / ms4 / 1e9, f * 8 / ms8 / 1e9);
  }
  for (int warps : {4, 8, 16}) {
    int threads = warps * 32;
    float ms = timeit([&] { dmma_kernel<<<sms, threads>>>(out, iters); });
    double f = 2.0 * 256 * 4 * 16 * (double)iters * sms * warps;  // 8x8x4 MACs per mma per warp
    printf("DMMA warps/SM=%2d  %.2f TF\n", warps, f / ms / 1e9);
  }
  return 0;
}
// mixed: even warps DFMA (ILP8), odd warps DMMA; reports each class's achieved rate
__global__ void mixed_kernel(double* out, int iters_f, int iters_m, unsigned long long* clk) {
  const int w = threadIdx.x / 32;
  long long t0 = clock64();
  if (w % 2 == 0) {
    double acc[8];
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_f; ++it)
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], 1.0000001, 1e-9);
    double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678) out[threadIdx.x] = s;
  } else {
    double a = threadIdx.x * 1e-3, b = 1.0001;
    double c[4][2] = {};
    for (int it = 0; it < iters_m; ++it)
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    double s = 0; for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[threadIdx.x] = s;
  }
  long long t1 = clock64();
  if (threadIdx.x % 32 == 0) clk[blockIdx.x * 64 + w] = t1 - t0;
}

int main2() {
  double* out; cudaMalloc(&out, 1 << 20);
  unsigned long long* clk; cudaMalloc(&clk, 148 * 64 * 8);
  int sms = 148, threads = 512;
  // balance: DFMA warp does 8*16*iters_f DFMA (=8*16*iters_f*64 FMA/warp at lane level: 32 lanes)
  for (int im : {0, 256, 512, 1024}) {
    int itf = 1024;
    float ms = timeit([&] { mixed_kernel<<<sms, threads>>>(out, itf, im, clk); });
    double dfma_flops = 2.0 * sms * (threads / 2) * itf * 16 * 8;
    double dmma_flops = 2.0 * 256 * 4 * 16 * (double)im * sms * (threads / 64);
    printf("mixed itf=%d itm=%d: %.3f ms  DFMA part %.2f TF  DMMA part %.2f TF  total %.2f TF\n", itf, im, ms,
           dfma_flops / ms / 1e9, dmma_flops / ms / 1e9, (dfma_flops + dmma_flops) / ms / 1e9);
  }
  return 0;
}
int main() { main1(); return main2(); }

// Which non-DFMA instruction classes cost the FP64 pipe throughput? 8 independent DFMA chains per
// thread with N instructions of one class after every 8 DFMAs, at 8 / 16 warps per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix2 fp64_mix2.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double ctab[64];

enum { LOP = 0, IMAD, MOV, SETP, SELP, LDS64, LDS128, FFMA, LDC, DADD, BRA, NCLS };
static const char* names[] = {"lop3", "imad", "mov", "setp", "selp(f)", "lds.64", "lds.128", "ffma", "ld.const", "dadd", "bra(uniform)"};

template <int CLS, int N>
__global__ void mix_kernel(double* out, int iters, double a, double b, int zero) {
  __shared__ double2 sm[1024];
  double acc[8];
  unsigned x[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  float f[4] = {1.f, 2.f, 3.f, 4.f};
  double dsum[4] = {0, 0, 0, 0};
  sm[threadIdx.x] = make_double2(threadIdx.x, 1.0);
  __syncthreads();
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(&sm[threadIdx.x & 511]);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const int c = j & 3;
        if (CLS == LOP) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(it), "r"(j + r));
        if (CLS == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(it), "r"(j + r));
        if (CLS == MOV) asm volatile("mov.b32 %0, %1;" : "=r"(x[c]) : "r"(it + j));
        if (CLS == SETP) asm volatile("{.reg .pred p; setp.lt.u32 p, %0, %1; @p add.u32 %0, %0, 1;}" : "+r"(x[c]) : "r"(it));
        if (CLS == SELP) asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.f32 %0, %0, 0f00000000, p;}" : "+f"(f[c]) : "r"(it | 1));
        if (CLS == LDS64) { double t; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(t) : "r"(sbase + 16 * ((j + r) & 15))); dsum[c] = t; }
        if (CLS == LDS128) { double t, t2; asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(t), "=d"(t2) : "r"(sbase + 16 * ((j + r) & 15))); dsum[c] = t; }
        if (CLS == FFMA) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(1.0001f), "f"(0.5f));
        if (CLS == LDC) { double t; asm volatile("ld.const.f64 %0, [%1];" : "=d"(t) : "l"((unsigned long long)(8 * ((it + j + r) & 63)) + (unsigned long long)zero)); dsum[c] = t; }
        if (CLS == DADD) asm volatile("add.f64 %0, %0, %1;" : "+d"(dsum[c]) : "d"(a));
        if (CLS == BRA) asm volatile("{.reg .pred p; setp.eq.u32 p, %0, 12345; @p bra L_%=; L_%=: }" :: "r"(zero + j));
      }
    }
  }
  double s = x[0] + x[1] + x[2] + x[3] + f[0] + f[1] + f[2] + f[3] + dsum[0] + dsum[1] + dsum[2] + dsum[3];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
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

template <int CLS, int N>
void run1(double* out) {
  const int sms = 148, iters = 2048;
  for (int warps : {8, 16}) {
    const int threads = warps * 32;
    float ms = timeit([&] { mix_kernel<CLS, N><<<sms, threads>>>(out, iters, 1.0000001, 1e-9, 0); });
    double f = 2.0 * sms * threads * (double)iters * 8 * 8;
    printf("  N=%-2d w%-2d %6.2f TF", N, warps, f / ms / 1e9);
  }
}
template <int CLS>
void run(double* out) {
  printf("%-12s", names[CLS]);
  run1<CLS, 2>(out); run1<CLS, 4>(out); run1<CLS, 8>(out); run1<CLS, 12>(out);
  printf("\n");
}

int main() {
  double* out; cudaMalloc(&out, 1 << 20);
  printf("DFMA TF/s (DFMA flops only) with N instructions of a class per 8 DFMAs\n");
  run<LOP>(out); run<IMAD>(out); run<MOV>(out); run<SETP>(out); run<SELP>(out); run<LDS64>(out);
  run<LDS128>(out); run<FFMA>(out); run<LDC>(out); run<DADD>(out); run<BRA>(out);
  return 0;
}
